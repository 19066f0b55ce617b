#!/bin/bash
# Round-2 closing session: GPU tests, bench line, reference arm, launch list, ncu captures.
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fresh_kernel|decode_kernel|score_kernel|select_|relevance|pack_kernel|retr_|qpack|lse_combine|out_combine" -c 300 --csv --log-file gpurun_out/final/launches.csv \
    python bench.py --profile --steps 2 --warmup 1 > gpurun_out/final/launch.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fresh_kernel -s 3 -c 1 \
    -o gpurun_out/final/fresh_full python bench.py --profile --steps 1 --warmup 1 > gpurun_out/final/ncu_fresh.log 2>&1; echo "ncu fresh rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 \
    -o gpurun_out/final/decode_full python tools/trace_decode.py long-video > gpurun_out/final/ncu_decode.log 2>&1; echo "ncu decode rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select_fast|relevance" -s 2 -c 2 \
    -o gpurun_out/final/sweep_select python tools/exp/sweep_select_one.py > gpurun_out/final/ncu_sel.log 2>&1; echo "ncu select rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:retr_out_kernel -s 1 -c 1 \
    -o gpurun_out/final/qattn python tools/exp/qattn_one.py > gpurun_out/final/ncu_qattn.log 2>&1; echo "ncu qattn rc=$?"
ls -la gpurun_out/final
