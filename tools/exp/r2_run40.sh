python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_fast -s 2 -c 1 -o gpurun_out/r02_select_sweep python tools/exp/select_one.py sweep > gpurun_out/ncu_sel.log 2>&1
tail -n 3 gpurun_out/ncu_sel.log
