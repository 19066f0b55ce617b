python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_decode_splits.py -q -x 2>&1 | tail -3
(timeout 200 python tools/trace_decode.py long-video
 timeout 200 python tools/trace_decode.py multi-turn
 timeout 300 python tools/exp/decode_bench.py base) > gpurun_out/r2_trace8.txt 2>&1
cat gpurun_out/r2_trace8.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 4 -c 1 -o gpurun_out/r2_ncu_decode python tools/exp/decode_one.py long-video 6 > gpurun_out/r2_ncu_decode.log 2>&1
tail -3 gpurun_out/r2_ncu_decode.log
