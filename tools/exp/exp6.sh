timeout 900 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -2
for B in 2 6 8; do timeout 120 python tools/exp_fused.py 32768 $B 20 2>&1 | grep -v "^$" | tail -1; done
timeout 120 python tools/exp_fused.py 24576 8 20 2>&1 | grep -v "^$" | tail -1
