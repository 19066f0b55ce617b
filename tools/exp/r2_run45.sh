python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:decode_kernel -s 20 -c 1 -o gpurun_out/r02_decode_cl python tools/exp/decode_one.py long-video 24 > gpurun_out/ncu_dcl.log 2>&1
tail -n 2 gpurun_out/ncu_dcl.log
