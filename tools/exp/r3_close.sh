#!/bin/bash
# Round-3 closing session (final sources): trap-build stability and compute-sanitizer on the
# fresh step / steady decode (incl. the SVL_DECODE_STATIC_PREFIX early path), then the
# r3_session captures (smoke, GPU tests, ncu, bench, reference arm, launch list, traces).
# The trap and trace variants are built before the call (build/trap, build/trace).
O=gpurun_out/r03; mkdir -p $O
: > $O/stability.txt
for c in toy nvila-4k long-video multi-turn; do
  SVL_LIB=build/trap/libsparsevila.so timeout 600 python tools/exp/many_calls.py $c 1000 >> $O/stability.txt 2>&1 || echo "$c: FAILED rc=$?" >> $O/stability.txt
done
cat $O/stability.txt
: > $O/sanitize.txt
for tool in memcheck racecheck synccheck; do
  for c in toy long-video; do
    echo "=== compute-sanitizer --tool $tool, $c, 2 calls" >> $O/sanitize.txt
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/exp/many_calls.py $c 2 > $O/san_${tool}_${c}.log 2>&1
    echo "rc=$?" >> $O/sanitize.txt
    tail -3 $O/san_${tool}_${c}.log >> $O/sanitize.txt
  done
done
cat $O/sanitize.txt
bash tools/exp/r3_session.sh
