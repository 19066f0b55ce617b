for i in 1 2; do python tools/exp/race.py multi-turn 40 2>&1 | grep -v "^$" | tail -1 | cut -c1-100; done
for i in 1 2; do SVL_NO_PDL=1 python tools/exp/race.py multi-turn 40 2>&1 | grep -v "^$" | tail -1 | cut -c1-100; done
python tools/exp/race.py long-video 40 2>&1 | grep -v "^$" | tail -1 | cut -c1-100
python tools/exp/race.py nvila-4k 40 2>&1 | grep -v "^$" | tail -1 | cut -c1-100
timeout 120 python tools/exp_fused.py 32768 8 20 2>&1 | grep -v "^$" | tail -1
timeout 120 python tools/exp_fused.py 32768 1 200 2>&1 | grep -v "^$" | tail -1
for i in 1 2; do timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1; done
