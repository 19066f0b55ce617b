python -c "import __graft_entry__ as g; g.build()" || exit 1
(timeout 200 python tools/trace_decode.py long-video; timeout 200 python tools/trace_decode.py multi-turn) > gpurun_out/r2_trace15.txt 2>&1
cat gpurun_out/r2_trace15.txt
