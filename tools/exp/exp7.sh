SVL_NO_PDL=1 timeout 300 compute-sanitizer --tool synccheck python tools/exp/one_mt.py 2>&1 | grep -v "^$" | head -6
for i in 1 2; do SVL_FRESH_CS=16 timeout 120 python tools/exp_fused.py 32768 8 20 2>&1 | grep -v "^$" | tail -1; done
SVL_FRESH_CS=16 timeout 120 python tools/exp_fused.py 24576 8 20 2>&1 | grep -v "^$" | tail -1
python tools/exp/race.py multi-turn 40 2>&1 | grep -v "^$" | tail -1
timeout 120 python tools/exp_fused.py 32768 1 200 2>&1 | grep -v "^$" | tail -1
for i in 1 2; do timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1; SVL_NO_PDL=1 timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1; done
