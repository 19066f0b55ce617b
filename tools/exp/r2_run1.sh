set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_gputest.txt
timeout 600 python bench.py > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err
tail -3 gpurun_out/r2_bench0.err
cat gpurun_out/r2_gputest.txt
