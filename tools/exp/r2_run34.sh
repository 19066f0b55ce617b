python -c "import __graft_entry__ as g; g.build()" || exit 1
SVL_VARIANT=pf16 SVL_DEFS="-DSVL_L2PF_STAGES=16" python -m paper_2510_17777_b200.build >/dev/null &
SVL_VARIANT=pf0 SVL_DEFS="-DSVL_L2PF_STAGES=0" python -m paper_2510_17777_b200.build >/dev/null &
wait
timeout 300 python tools/exp/fresh_bench.py base
SVL_LIB=build/pf16/libsparsevila.so timeout 300 python tools/exp/fresh_bench.py pf16
SVL_LIB=build/pf0/libsparsevila.so timeout 300 python tools/exp/fresh_bench.py pf0
