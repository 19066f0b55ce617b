for i in 1 2; do timeout 60 python tools/exp_fused.py 32768 1 300 2>&1 | grep -v "^$" | tail -1 | cut -c1-90; SVL_LIB=build/nopf/libsparsevila.so timeout 60 python tools/exp_fused.py 32768 1 300 2>&1 | grep -v "^$" | tail -1 | cut -c1-90; done
timeout 60 python tools/exp_fused.py 4096 1 300 2>&1 | grep -v "^$" | tail -1 | cut -c1-90
for i in 1 2; do SVL_FRESH_CS=16 timeout 60 python tools/exp_fused.py 32768 8 20 2>&1 | grep -v "^$" | tail -1 | cut -c1-90; done
SVL_FRESH_CS=8 timeout 60 python tools/exp/race.py multi-turn 40 2>&1 | grep -v "^$" | tail -1 | cut -c1-100
timeout 60 python tools/exp/race.py long-video 40 2>&1 | grep -v "^$" | tail -1 | cut -c1-100
timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
