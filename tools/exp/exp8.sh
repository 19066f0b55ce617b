for i in 1 2 3 4; do python tools/exp/race.py multi-turn 40 2>&1 | grep -v "^$" | tail -1 | cut -c1-80; done
echo NO_PDL
for i in 1 2 3 4; do SVL_NO_PDL=1 python tools/exp/race.py multi-turn 40 2>&1 | grep -v "^$" | tail -1 | cut -c1-80; done
echo DRAIN
for i in 1 2 3 4; do SVL_LIB=build/drain/libsparsevila.so python tools/exp/race.py multi-turn 40 2>&1 | grep -v "^$" | tail -1 | cut -c1-80; done
