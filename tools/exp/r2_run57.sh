#!/bin/bash
for v in head new mode0r head new mode0r; do
  if [ $v = new ]; then L=paper_2510_17777_b200/libsparsevila.so; else L=build/$v/libsparsevila.so; fi
  SVL_LIB=$L timeout 300 python tools/exp/twocall_bench.py $v 2>&1 | tail -3
  SVL_LIB=$L timeout 300 python tools/exp/fresh_bench.py $v 2>&1 | tail -2
done
