python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/exp/fresh_bench.py base 2>&1 | tail -3
SVL_LIB=build/trace/libsparsevila.so python tools/trace_fresh.py long-video > gpurun_out/trace_fresh_base.txt 2>&1
cat gpurun_out/trace_fresh_base.txt
