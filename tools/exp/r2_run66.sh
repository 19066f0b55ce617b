#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_decode_splits.py tests/test_gpu_parity.py tests/test_gpu_push.py tests/test_gpu_seqpar.py tests/test_gpu_pack.py -x -q 2>&1 | tail -3
for v in cpasync new cpasync new; do
  if [ $v = new ]; then L=paper_2510_17777_b200/libsparsevila.so; else L=build/$v/libsparsevila.so; fi
  SVL_LIB=$L timeout 300 python tools/exp/decode_bench.py $v 2>&1 | tail -4
  SVL_LIB=$L timeout 300 python tools/exp/twocall_bench.py $v 2>&1 | tail -3
done
