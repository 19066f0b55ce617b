# usage: bash tools/exp/r3_ab.sh "p0 p1 ..." "t0 t1 ..."  (variant dirs under build/)
P="$1"; T="$2"
for rep in 1 2; do for v in $P; do SVL_LIB=build/$v/libsparsevila.so CFGS=long-video python tools/exp/fresh_bench.py $v 2>&1 | grep long-video; done; done
for v in $T; do echo "== $v"; SVL_LIB=build/$v/libsparsevila.so python tools/trace_fresh.py long-video 2>&1 | head -32; done
