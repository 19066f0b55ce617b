python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_decode_splits.py tests/test_gpu_parity.py tests/test_gpu_push.py tests/test_gpu_pack.py -x -q 2>&1 | tail -8 > gpurun_out/r2_t5.txt
(timeout 200 python tools/trace_decode.py long-video
 timeout 200 python tools/trace_decode.py nvila-4k
 timeout 200 python tools/trace_decode.py multi-turn
 timeout 300 python tools/exp/decode_bench.py base) > gpurun_out/r2_trace5.txt 2>&1
cat gpurun_out/r2_t5.txt gpurun_out/r2_trace5.txt
