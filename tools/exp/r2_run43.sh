python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2_bench6.json 2> gpurun_out/r2_bench6.err; tail -n 2 gpurun_out/r2_bench6.err
python -c "
import json; d=json.load(open('gpurun_out/r2_bench6.json'))
print(d['us_per_layer'], d['steady'], d['throughput_sweep']['us_per_layer'], json.dumps(d['configs']), d['cold_single_layer_us'])"
