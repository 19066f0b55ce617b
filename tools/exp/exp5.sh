for B in 5 6 7; do python tools/exp/fresh_one.py 32768 $B 2 2 2>&1 | grep -v "^$" | tail -1; done
python tools/exp/fresh_one.py 24576 8 2 2 2>&1 | grep -v "^$" | tail -1
python tools/exp/fresh_one.py 32768 8 1 1 2>&1 | grep -v "^$" | tail -1
dmesg 2>&1 | tail -15
