SVL_LIB=build/trace/libsparsevila.so python tools/trace_fresh.py long-video 2>&1 | head -${1:-60}
