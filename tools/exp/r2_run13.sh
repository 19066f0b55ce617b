python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_decode_splits.py tests/test_gpu_parity.py tests/test_gpu_push.py tests/test_gpu_pack.py tests/test_gpu_fused.py -x -q 2>&1 | tail -4
(timeout 200 python tools/trace_decode.py long-video
 timeout 300 python tools/exp/decode_bench.py base) > gpurun_out/r2_trace13.txt 2>&1
cat gpurun_out/r2_trace13.txt
