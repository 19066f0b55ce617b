python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 20 -c 1 -o gpurun_out/r2_ncu_decode2 python tools/exp/decode_one.py long-video 24 > gpurun_out/r2_ncu_decode2.log 2>&1
tail -2 gpurun_out/r2_ncu_decode2.log
