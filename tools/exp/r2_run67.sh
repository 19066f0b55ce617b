#!/bin/bash
for v in new t384d3 t256d3 t384 new t384d3 t256d3 t384; do
  if [ $v = new ]; then L=paper_2510_17777_b200/libsparsevila.so; else L=build/$v/libsparsevila.so; fi
  SVL_LIB=$L timeout 300 python tools/exp/twocall_bench.py $v 2>&1 | tail -3
done
