python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python bench.py --mode seq-split --steps 20 --warmup 3 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2_bench5.json 2> gpurun_out/r2_bench5.err; tail -3 gpurun_out/r2_bench5.err
python -c "
import json; d=json.load(open('gpurun_out/r2_bench5.json'))
print(json.dumps(d['page_retrieval'])); print(json.dumps(d['prefill'])[:1500])"
