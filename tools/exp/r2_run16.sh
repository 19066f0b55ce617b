python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
(timeout 200 python tools/trace_decode.py long-video; timeout 200 python tools/trace_decode.py multi-turn; timeout 300 python tools/exp/decode_bench.py base) > gpurun_out/r2_trace16.txt 2>&1
cat gpurun_out/r2_trace16.txt
