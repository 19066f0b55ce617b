python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_decode_splits.py -q -x 2>&1 | tail -3
(timeout 200 python tools/trace_decode.py long-video
 timeout 300 python tools/exp/decode_bench.py base) > gpurun_out/r2_trace10.txt 2>&1
cat gpurun_out/r2_trace10.txt
