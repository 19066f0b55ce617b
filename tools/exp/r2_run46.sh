python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_retrieve_tc.py tests/test_gpu_decode_splits.py -q -x 2>&1 | tail -3
timeout 300 python tools/exp/decode_bench.py pad33 2>&1 | head -3
