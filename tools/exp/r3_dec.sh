timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode_splits.py tests/test_gpu_push.py tests/test_gpu_pack.py -x -q 2>&1 | tail -3
for L in dold cur; do SVL_LIB=build/$L/libsparsevila.so DCFGS="long-video:0,16;nvila-4k:0;multi-turn:0;sweep:0" python tools/exp/decode_bench.py $L 2>&1 | grep -v "^lib"; done
SVL_LIB=build/trace/libsparsevila.so python tools/trace_decode.py long-video 2>&1 | tail -9
