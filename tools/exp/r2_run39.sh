python -c "import __graft_entry__ as g; g.build()" || exit 1
SVL_VARIANT=sel4k SVL_DEFS="-DSVL_SELECT_ROWS_PER_CTA=4096" python -m paper_2510_17777_b200.build >/dev/null &
SVL_VARIANT=sel8k SVL_DEFS="-DSVL_SELECT_ROWS_PER_CTA=8192" python -m paper_2510_17777_b200.build >/dev/null &
wait
timeout 300 python tools/exp/twocall_bench.py base
SVL_LIB=build/sel4k/libsparsevila.so timeout 300 python tools/exp/twocall_bench.py sel4k
SVL_LIB=build/sel8k/libsparsevila.so timeout 300 python tools/exp/twocall_bench.py sel8k
