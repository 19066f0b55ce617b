python -c "import __graft_entry__ as g; g.build()" || exit 1
SVL_VARIANT=pvold SVL_DEFS="-DSVL_PV_ROWS=0" python -m paper_2510_17777_b200.build >/dev/null
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_fused_ties.py -q -x 2>&1 | tail -2
timeout 300 python tools/exp/fresh_bench.py pvrows
SVL_LIB=build/pvold/libsparsevila.so timeout 300 python tools/exp/fresh_bench.py pvold
timeout 300 python tools/trace_fresh.py long-video | head -14
