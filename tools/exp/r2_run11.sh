python -c "import __graft_entry__ as g; g.build()" || exit 1
SVL_VARIANT=nomerge SVL_DEFS="-DSVL_EXP_NOMERGE=1" python -m paper_2510_17777_b200.build >/dev/null &
SVL_VARIANT=nocomp SVL_DEFS="-DSVL_EXP_NOCOMPUTE=1 -DSVL_EXP_NOMERGE=1" python -m paper_2510_17777_b200.build >/dev/null &
SVL_VARIANT=nbuf2 SVL_DEFS="-DSVL_DECODE_NBUF=2" python -m paper_2510_17777_b200.build >/dev/null &
wait
(SVL_LIB=build/nomerge/libsparsevila.so timeout 300 python tools/exp/decode_bench.py nomerge
 SVL_LIB=build/nocomp/libsparsevila.so timeout 300 python tools/exp/decode_bench.py nocompute+nomerge
 SVL_LIB=build/nbuf2/libsparsevila.so timeout 300 python tools/exp/decode_bench.py nbuf2) > gpurun_out/r2_exp11.txt 2>&1
cat gpurun_out/r2_exp11.txt
