python -c "import __graft_entry__ as g; g.build()" || exit 1
SVL_VARIANT=trace SVL_DEFS="-DSVL_TRACE_BUILD=1" python -m paper_2510_17777_b200.build >/dev/null
SVL_VARIANT=tracenf SVL_DEFS="-DSVL_TRACE_BUILD=1 -DSVL_EXP_NOFINAL=1" python -m paper_2510_17777_b200.build >/dev/null
timeout 300 python -m pytest tests/test_gpu_decode_splits.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
(SVL_LIB=build/trace/libsparsevila.so timeout 200 python tools/trace_decode.py long-video
 SVL_LIB=build/tracenf/libsparsevila.so timeout 200 python tools/trace_decode.py long-video
 timeout 300 python tools/exp/decode_bench.py base) > gpurun_out/r2_trace19.txt 2>&1
cat gpurun_out/r2_trace19.txt
