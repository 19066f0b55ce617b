python -c "import __graft_entry__ as g; g.build()" || exit 1
(timeout 200 python tools/trace_decode.py long-video
 timeout 200 python tools/trace_decode.py nvila-4k
 timeout 300 python tools/exp/decode_bench.py base) > gpurun_out/r2_trace9.txt 2>&1
cat gpurun_out/r2_trace9.txt
