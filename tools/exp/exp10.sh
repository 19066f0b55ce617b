for v in default V1 V2 drain; do
  L=build/$v/libsparsevila.so; [ $v = default ] && L=paper_2510_17777_b200/libsparsevila.so
  for i in 1 2; do SVL_LIB=$L timeout 120 python tools/exp_fused.py 32768 1 300 2>&1 | grep -v "^$" | tail -1 | cut -c1-90; done
done
