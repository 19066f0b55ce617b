"""One sweep layer's svl_retrieve (score + relevance + select) for ncu."""
import sys, torch
sys.path.insert(0, ".")
from paper_2510_17777_b200 import svl, inputs as gen
wl = gen.CONFIGS["sweep"]
x = gen.make_decode_inputs(wl, seed=1, device="cuda")
ws = svl.Workspace()
for _ in range(3):
    svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws)
torch.cuda.synchronize()
print("ok")
