#!/bin/bash
for v in rel4w new sl4k rel4w new sl4k; do
  if [ $v = new ]; then L=paper_2510_17777_b200/libsparsevila.so; else L=build/$v/libsparsevila.so; fi
  SVL_LIB=$L timeout 300 python tools/exp/twocall_bench.py $v 2>&1 | tail -3 | head -1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
