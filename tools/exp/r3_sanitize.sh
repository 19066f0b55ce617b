python -c "import __graft_entry__ as g; g.build()" || exit 1
SVL_VARIANT=trap SVL_DEFS="-DSVL_DEBUG_TRAP=1" python -m paper_2510_17777_b200.build > /dev/null || exit 1
OUT=gpurun_out/sanitize_r03.txt
: > $OUT
for c in toy nvila-4k long-video multi-turn; do
  SVL_LIB=build/trap/libsparsevila.so timeout 600 python tools/exp/many_calls.py $c 1000 >> $OUT 2>&1 || echo "$c: FAILED rc=$?" >> $OUT
done
for tool in memcheck racecheck synccheck; do
  for c in toy nvila-4k long-video; do
    echo "=== compute-sanitizer --tool $tool, $c, 3 calls" >> $OUT
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/exp/many_calls.py $c 3 > gpurun_out/san_${tool}_${c}.log 2>&1
    echo "rc=$?" >> $OUT
    tail -4 gpurun_out/san_${tool}_${c}.log >> $OUT
  done
done
cat $OUT
