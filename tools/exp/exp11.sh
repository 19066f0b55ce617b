for i in 1 2 3; do timeout 120 python tools/exp_fused.py 32768 1 300 2>&1 | grep -v "^$" | tail -1 | cut -c1-90; SVL_LIB=build/nopf/libsparsevila.so timeout 120 python tools/exp_fused.py 32768 1 300 2>&1 | grep -v "^$" | tail -1 | cut -c1-90; done
for i in 1 2; do SVL_FRESH_CS=16 timeout 120 python tools/exp_fused.py 32768 8 20 2>&1 | grep -v "^$" | tail -1 | cut -c1-90; done
SVL_FRESH_CS=8 python tools/exp/race.py multi-turn 40 2>&1 | grep -v "^$" | tail -1 | cut -c1-100
python tools/exp/race.py long-video 40 2>&1 | grep -v "^$" | tail -1 | cut -c1-100
