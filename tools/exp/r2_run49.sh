#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_question_attention.py -x -q 2>&1 | tail -4
echo "== P in TMEM (default)"; timeout 600 python tools/exp/qattn_bench.py 2>&1 | tail -4
echo "== P in smem"; SVL_LIB=build/psmem/libsparsevila.so timeout 600 python tools/exp/qattn_bench.py 2>&1 | tail -4
