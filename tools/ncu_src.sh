set -x
python - <<'PY'
PY
ncu --clock-control none --import-source on --set full -k regex:fresh_kernel -s 3 -c 1 -o gpurun_out/fresh_src python tools/exp_fused.py 32768 1 3 > gpurun_out/ncu_src.log 2>&1
ncu -i gpurun_out/fresh_src.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/fresh_src_source.csv 2>&1
ls -la gpurun_out/
