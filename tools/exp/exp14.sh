for i in 1 2; do timeout 60 python tools/exp_fused.py 32768 1 300 2>&1 | grep -v "^$" | tail -1 | cut -c1-90; done
timeout 60 python tools/exp/race.py multi-turn 40 2>&1 | grep -v "^$" | tail -1 | cut -c1-100
timeout 60 python tools/exp/race.py long-video 40 2>&1 | grep -v "^$" | tail -1 | cut -c1-100
for i in 1 2; do timeout 400 python -m pytest tests -m gpu -q 2>&1 | tail -1; done
python tools/trace_fresh.py 2>&1 | head -14
