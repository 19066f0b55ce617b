#!/bin/bash
mkdir -p gpurun_out
for v in vpf0 default vpf300 vpf100 vpf0 default vpf300 vpf100; do
  if [ $v = default ]; then L=paper_2510_17777_b200/libsparsevila.so; else L=build/$v/libsparsevila.so; fi
  SVL_LIB=$L timeout 300 python tools/exp/fresh_bench.py $v 2>&1 | tail -2
done
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_fused_ties.py -x -q 2>&1 | tail -2
