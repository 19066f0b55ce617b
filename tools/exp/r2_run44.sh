python -c "import __graft_entry__ as g; g.build()" || exit 1
(timeout 200 python tools/trace_decode.py long-video; timeout 200 python tools/trace_decode.py nvila-4k; timeout 200 python tools/trace_decode.py multi-turn) 2>&1
