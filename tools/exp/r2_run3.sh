python -c "import __graft_entry__ as g; g.build()" || exit 1
SVL_VARIANT=nocoop SVL_DEFS="-DSVL_DECODE_NO_COOP=1" python -m paper_2510_17777_b200.build >/dev/null &
SVL_VARIANT=nopdl SVL_DEFS="-DSVL_DECODE_NO_PDL=1" python -m paper_2510_17777_b200.build >/dev/null &
SVL_VARIANT=occ1 SVL_DEFS="-DSVL_DECODE_OCC=1" python -m paper_2510_17777_b200.build >/dev/null &
wait
(timeout 300 python tools/exp/decode_bench.py base
 SVL_LIB=build/nocoop/libsparsevila.so timeout 300 python tools/exp/decode_bench.py nocoop
 SVL_LIB=build/nopdl/libsparsevila.so timeout 300 python tools/exp/decode_bench.py nopdl
 SVL_LIB=build/occ1/libsparsevila.so timeout 300 python tools/exp/decode_bench.py occ1) > gpurun_out/r2_decode_sweep.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_fused_ties.py -q 2>&1 | tail -5 >> gpurun_out/r2_decode_sweep.txt
cat gpurun_out/r2_decode_sweep.txt
