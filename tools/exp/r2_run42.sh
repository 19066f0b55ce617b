python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_decode_splits.py tests/test_gpu_parity.py tests/test_gpu_push.py tests/test_gpu_pack.py tests/test_gpu_seqpar.py -q -x 2>&1 | tail -3
timeout 300 python tools/exp/decode_bench.py base
