python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/exp/fresh_bench.py base
timeout 300 python tools/trace_fresh.py long-video | grep -A5 "end of the stream\|phase end"
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_fused_ties.py -q -x 2>&1 | tail -2
