import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
name = sys.argv[1] if len(sys.argv) > 1 else "multi-turn"
wl = gen.CONFIGS[name]
x = gen.make_decode_inputs(wl, seed=31, device="cuda")
torch.cuda.synchronize()
out, idx = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k)
torch.cuda.synchronize()
print("done", idx.sum().item())
