timeout 60 python tools/exp_fused.py 32768 8 20 2>&1 | grep -v "^$" | tail -1 | cut -c1-90
timeout 60 python tools/exp_fused.py 32768 1 300 2>&1 | grep -v "^$" | tail -1 | cut -c1-90
for i in 1 2; do timeout 60 python tools/exp/race.py multi-turn 40 2>&1 | grep -v "^$" | tail -1 | cut -c1-100; done
for i in 1 2 3; do timeout 400 python -m pytest tests -m gpu -q 2>&1 | tail -1; done
SVL_NO_PDL=1 timeout 400 python -m pytest tests -m gpu -q 2>&1 | tail -1
