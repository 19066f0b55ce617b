python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/exp/twocall_bench.py unr4
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
