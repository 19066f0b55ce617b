#!/bin/bash
set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_question_attention.py -x -q 2>&1 | tail -25
