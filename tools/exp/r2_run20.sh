python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err
python -c "
import json; d=json.load(open('gpurun_out/r2_bench2.json'))
print(d['us_per_layer'], d['steady'], d['unfused_us_per_layer'], d['throughput_sweep'], d['pack_once'], d['e2e']['ms_per_step'], d['clocks'])"
