#!/bin/bash
# Round-3 session: build + smoke, GPU tests, ncu capture of fresh_kernel (-> traffic file keyed
# to the source), bench line, reference arm, launch list, decode capture.
O=gpurun_out/r03; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/gputests.txt; cat $O/gputests.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fresh_kernel -s 3 -c 1 \
    -o $O/fresh_full python bench.py --profile --steps 1 --warmup 1 > $O/ncu_fresh.log 2>&1; echo "ncu fresh rc=$?"
python tools/fresh_traffic_json.py $O/fresh_full.ncu-rep "profiles/ncu_r03_fresh_kernel.txt" > $O/traffic.json 2>&1; cat $O/traffic.json
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fresh_kernel|decode_kernel|score_kernel|select_|relevance|pack_kernel|retr_|qpack|lse_combine|out_combine" -c 300 --csv --log-file $O/launches.csv \
    python bench.py --profile --steps 2 --warmup 1 > $O/launch.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 \
    -o $O/decode_full python tools/trace_decode.py long-video > $O/ncu_decode.log 2>&1; echo "ncu decode rc=$?"
SVL_LIB=build/trace/libsparsevila.so python tools/trace_fresh.py long-video > $O/trace_fresh.txt 2>&1
ls -la $O
