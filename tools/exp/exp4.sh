python tools/exp/fresh_one.py 32768 8 1 1 2>&1 | grep -v "^$" | tail -1
python tools/exp/fresh_one.py 32768 8 3 3 2>&1 | grep -v "^$" | tail -1
SVL_NO_PDL=1 python tools/exp/fresh_one.py 32768 8 3 3 2>&1 | grep -v "^$" | tail -1
python tools/exp/fresh_one.py 32768 4 3 3 2>&1 | grep -v "^$" | tail -1
python tools/exp/fresh_one.py 32768 3 3 3 2>&1 | grep -v "^$" | tail -1
timeout 600 compute-sanitizer --tool memcheck python tools/exp/fresh_one.py 32768 8 1 1 2>&1 | grep -v "^$" | head -30
