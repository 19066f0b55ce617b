#!/bin/bash
mkdir -p gpurun_out
SVL_LIB=build/mode0/libsparsevila.so timeout 300 python tools/exp/twocall_bench.py mode0 2>&1 | tail -3
timeout 300 python tools/exp/twocall_bench.py split3 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_retrieve_tc.py -x -q 2>&1 | tail -3
