python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python bench.py > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err; tail -3 gpurun_out/r2_bench3.err
timeout 900 python bench.py --mode sweep-heads --fused-gather --steps 20 --warmup 3 > gpurun_out/r2_sweepheads1.json 2> gpurun_out/r2_sweepheads1.err; tail -3 gpurun_out/r2_sweepheads1.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; tail -2 gpurun_out/r2_ref.err
cat gpurun_out/r2_sweepheads1.json gpurun_out/r2_ref.json
