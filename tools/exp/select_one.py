"""A few two-call retrieves on the sweep config (for ncu on the selection kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
name = sys.argv[1] if len(sys.argv) > 1 else "sweep"
wl = gen.CONFIGS[name]
x = gen.make_decode_inputs(wl, seed=1, device="cuda")
ws = svl.Workspace()
for _ in range(3):
    svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws)
torch.cuda.synchronize()
