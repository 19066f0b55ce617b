python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
OUT=gpurun_out/sanitize_r02b.txt
: > $OUT
for tool in memcheck racecheck synccheck; do
  for c in toy nvila-4k; do
    echo "=== compute-sanitizer --tool $tool, $c, 3 calls" >> $OUT
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/exp/many_calls.py $c 3 > gpurun_out/san2_${tool}_${c}.log 2>&1
    echo "rc=$?" >> $OUT
    tail -3 gpurun_out/san2_${tool}_${c}.log >> $OUT
  done
done
for c in long-video multi-turn; do
  echo "=== compute-sanitizer --tool memcheck, $c, 1 call" >> $OUT
  timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/exp/many_calls.py $c 1 > gpurun_out/san2_memcheck_${c}.log 2>&1
  echo "rc=$?" >> $OUT
  tail -3 gpurun_out/san2_memcheck_${c}.log >> $OUT
done
cat $OUT
