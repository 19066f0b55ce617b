#!/bin/bash
SVL_LIB=build/st2/libsparsevila.so timeout 300 python tools/exp/stage2_probe.py
timeout 300 python tools/exp/twocall_bench.py refine 2>&1 | tail -3
timeout 300 python tools/exp/fresh_bench.py refine 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_fused_ties.py tests/test_gpu_retrieve_tc.py -x -q 2>&1 | tail -3
