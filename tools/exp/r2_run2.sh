set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_decode_splits.py -x -q 2>&1 | tail -25 > gpurun_out/r2_t_splits.txt
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r2_gputest2.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
cat gpurun_out/r2_t_splits.txt gpurun_out/r2_gputest2.txt gpurun_out/r2_smoke.txt; tail -5 gpurun_out/r2_bench1.err
