#!/bin/bash
mkdir -p gpurun_out/sanitize2
OUT=gpurun_out/sanitize2/summary.txt
: > $OUT
echo "=== path check (A/B build: flag 0x200 = refinement round ran, 0x100 = generic fallback)" >> $OUT
SVL_LIB=build/st2/libsparsevila.so timeout 300 python tools/exp/sanitize_new.py 1 >> $OUT 2>&1
echo "=== 200 back-to-back calls (product build)" >> $OUT
timeout 600 python tools/exp/sanitize_new.py 200 >> $OUT 2>&1
for tool in memcheck racecheck synccheck; do
  echo "=== compute-sanitizer --tool $tool, 2 calls" >> $OUT
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/exp/sanitize_new.py 2 > gpurun_out/sanitize2/${tool}.log 2>&1
  echo "rc=$?" >> $OUT
  tail -3 gpurun_out/sanitize2/${tool}.log >> $OUT
done
cat $OUT
