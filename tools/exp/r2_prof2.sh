python -c "import __graft_entry__ as g; g.build()" || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fresh_kernel|decode_kernel|score_kernel|select_|pack_kernel" -c 200 --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --profile --steps 2 --warmup 1 > gpurun_out/launch.log 2>&1
tail -n 2 gpurun_out/launch.log
