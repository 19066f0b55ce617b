#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/exp/qattn_bench.py 2>&1 | tail -8
