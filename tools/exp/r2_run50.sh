#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench_r02b.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r02b.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "unit", "ms_per_step", "gpu_launches")})
print("roofline", d["roofline"])
print("e2e", d["e2e"])
for r in d["extra"]["question_retrieve"]["runs"] if "extra" in d else d.get("question_retrieve", {}).get("runs", []):
    print(r)
PY
