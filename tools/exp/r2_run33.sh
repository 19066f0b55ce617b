python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/trace_fresh.py long-video > gpurun_out/trace_r02_fresh.txt 2>&1
cat gpurun_out/trace_r02_fresh.txt
