mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -3
SVL_LIB=build/rf/libsparsevila.so timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -2
for r in 1 2; do
for v in head rf; do SVL_LIB=build/$v/libsparsevila.so timeout 120 python tools/exp_fused.py 32768 1 200; done
timeout 120 python tools/exp_fused.py 32768 1 200
done
python tools/trace_fresh.py 2>&1 | head -14
SVL_LIB=build/rf/libsparsevila.so python tools/trace_fresh.py 2>&1 | head -30
