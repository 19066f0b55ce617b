#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_fast|relevance" -s 2 -c 2 -o gpurun_out/sweep_sel2 python tools/exp/sweep_select_one.py > gpurun_out/sweep_sel2.log 2>&1
tail -1 gpurun_out/sweep_sel2.log
