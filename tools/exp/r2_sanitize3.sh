python -c "import __graft_entry__ as g; g.build()" || exit 1
SVL_VARIANT=trap SVL_DEFS="-DSVL_DEBUG_TRAP=1" python -m paper_2510_17777_b200.build > /dev/null || exit 1
OUT=gpurun_out/sanitize_r02c.txt
: > $OUT
for c in toy nvila-4k long-video multi-turn; do
  SVL_LIB=build/trap/libsparsevila.so timeout 600 python tools/exp/many_calls.py $c 1000 >> $OUT 2>&1 || echo "$c: FAILED rc=$?" >> $OUT
done
for tool in memcheck racecheck synccheck; do
  for c in toy nvila-4k long-video; do
    echo "=== compute-sanitizer --tool $tool, $c, 2 calls" >> $OUT
    timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/exp/many_calls.py $c 2 > gpurun_out/san3_${tool}_${c}.log 2>&1
    echo "rc=$?" >> $OUT
    tail -2 gpurun_out/san3_${tool}_${c}.log >> $OUT
  done
done
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2 >> $OUT
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2_bench4.json 2> gpurun_out/r2_bench4.err
python -c "import json; d=json.load(open('gpurun_out/r2_bench4.json')); print(d['us_per_layer'], d['steady']['us_per_layer'])" >> $OUT
cat $OUT
