python -c "import __graft_entry__ as g; g.build()" || exit 1
SVL_VARIANT=oneexp SVL_DEFS="-DSVL_LSE_ONE_EXP=1" python -m paper_2510_17777_b200.build >/dev/null
SVL_VARIANT=traceone SVL_DEFS="-DSVL_LSE_ONE_EXP=1 -DSVL_TRACE_BUILD=1" python -m paper_2510_17777_b200.build >/dev/null
timeout 300 python tools/exp/fresh_bench.py base
SVL_LIB=build/oneexp/libsparsevila.so timeout 300 python tools/exp/fresh_bench.py oneexp
SVL_LIB=build/traceone/libsparsevila.so timeout 300 python tools/trace_fresh.py long-video | grep -A5 "end of the stream\|phase end" 
