# One GPU session: bench line, reference arm, ncu launch list and full captures.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile --steps 2 --warmup 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fresh_kernel -s 3 -c 1 \
    -o gpurun_out/fresh_full python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_fresh.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 \
    -o gpurun_out/decode_full python tools/trace_decode.py long-video > gpurun_out/ncu_decode.log 2>&1
ls -la gpurun_out
