#!/bin/bash
for v in new nb1 nb1o3 new nb1 nb1o3; do
  if [ $v = new ]; then L=paper_2510_17777_b200/libsparsevila.so; else L=build/$v/libsparsevila.so; fi
  SVL_LIB=$L timeout 300 python tools/exp/twocall_bench.py $v 2>&1 | tail -3
done
SVL_LIB=build/nb1/libsparsevila.so timeout 900 python -m pytest tests/test_gpu_decode_splits.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
