SVL_LIB=build/st2/libsparsevila.so timeout 300 python tools/exp/stage2_probe.py
