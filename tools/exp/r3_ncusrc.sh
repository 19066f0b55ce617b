python -c "import __graft_entry__ as g; g.build()" || exit 1
ncu --clock-control none --import-source on --set full --warp-sampling-interval 0 --warp-sampling-buffer-size 536870912 -k regex:fresh_kernel -s 3 -c 1 -o gpurun_out/fresh_src python tools/exp/fresh_one.py 32768 1 5 > gpurun_out/ncu_src.log 2>&1
ncu -i gpurun_out/fresh_src.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/fresh_src_source.csv 2>&1
ncu -i gpurun_out/fresh_src.ncu-rep --page source --csv --print-source cuda > gpurun_out/fresh_src_cuda.csv 2>&1
tail -3 gpurun_out/ncu_src.log
