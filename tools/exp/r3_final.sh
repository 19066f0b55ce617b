#!/bin/bash
# Round-3 closing session: trap-build stability, GPU tests, ncu capture (traffic keyed to the
# source), bench line, reference arm, launch list, decode capture, phase trace.
O=gpurun_out/r03; mkdir -p $O
: > $O/stability.txt
for c in toy nvila-4k long-video multi-turn; do
  SVL_LIB=build/trap/libsparsevila.so timeout 600 python tools/exp/many_calls.py $c 1000 >> $O/stability.txt 2>&1 || echo "$c: FAILED rc=$?" >> $O/stability.txt
done
cat $O/stability.txt
bash tools/exp/r3_session.sh
