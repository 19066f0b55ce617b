for v in prest default; do
  L=build/$v/libsparsevila.so; [ $v = default ] && L=paper_2510_17777_b200/libsparsevila.so
  echo "== $v"
  SVL_LIB=$L timeout 500 compute-sanitizer --tool memcheck --print-limit 3 python -m pytest tests/test_gpu_fused.py -q -k "configs and multi" 2>&1 | grep -E "passed|failed|ParityError|ERROR SUMMARY" | head -4
done
