timeout 600 python -m pytest tests/test_gpu_fused.py -q -rf 2>&1 | tail -8
for r in 1 2 3; do timeout 120 python tools/exp_fused.py 32768 1 200; SVL_LIB=build/rf/libsparsevila.so timeout 120 python tools/exp_fused.py 32768 1 200 2>&1 | tail -1; done
