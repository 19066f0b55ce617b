"""Repeat svl_fresh_decode_step on fixed inputs; count runs whose idx/out differ from run 0."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
name = sys.argv[1] if len(sys.argv) > 1 else "multi-turn"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
wl = gen.CONFIGS[name]
x = gen.make_decode_inputs(wl, seed=31, device="cuda")
ref = None
bad_i = bad_o = 0
units = set()
for r in range(reps):
    out, idx = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k)
    torch.cuda.synchronize()
    if ref is None:
        ref = (out.clone(), idx.clone())
        continue
    if not torch.equal(idx, ref[1]):
        bad_i += 1
        d = (idx != ref[1]).any(-1).nonzero().tolist()
        units.update(tuple(t) for t in d)
    if not torch.equal(out, ref[0]):
        bad_o += 1
print(f"{os.environ.get('SVL_LIB', 'default')} {name}: {reps} runs, idx differs in {bad_i}, out in {bad_o}; units {sorted(units)[:10]}")
