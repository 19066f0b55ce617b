python -c "import __graft_entry__ as g; g.build()" || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --profile --steps 2 --warmup 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fresh_kernel -s 3 -c 1 \
    -o gpurun_out/r02_fresh_full python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_fresh.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 20 -c 1 \
    -o gpurun_out/r02_decode_full python tools/exp/decode_one.py long-video 24 > gpurun_out/ncu_decode.log 2>&1
tail -2 gpurun_out/ncu_fresh.log gpurun_out/ncu_decode.log
