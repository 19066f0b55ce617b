for i in 1 2 3; do timeout 120 python tools/exp_fused.py 32768 2 20 2>&1 | grep -v "^$" | tail -1; done
timeout 120 python tools/exp_fused.py 32768 8 20 2>&1 | grep -v "^$" | tail -1
timeout 120 python tools/exp_fused.py 32768 1 200 2>&1 | grep -v "^$" | tail -1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
