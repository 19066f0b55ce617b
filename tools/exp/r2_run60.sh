#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_fused_ties.py tests/test_gpu_retrieve_tc.py tests/test_gpu_pages.py tests/test_gpu_seqpar.py -x -q 2>&1 | tail -3
for v in head new head new; do
  if [ $v = new ]; then L=paper_2510_17777_b200/libsparsevila.so; else L=build/$v/libsparsevila.so; fi
  SVL_LIB=$L timeout 300 python tools/exp/twocall_bench.py $v 2>&1 | tail -3
  SVL_LIB=$L timeout 300 python tools/exp/fresh_bench.py $v 2>&1 | tail -2
done
