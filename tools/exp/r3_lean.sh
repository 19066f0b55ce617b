timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_fused_ties.py -x -q 2>&1 | tail -15
CFGS=long-video,nvila-4k python tools/exp/fresh_bench.py lean 2>&1 | tail -3
SVL_LIB=build/trace/libsparsevila.so python tools/trace_fresh.py long-video 2>&1 | head -60
