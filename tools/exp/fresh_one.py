import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
nv = int(sys.argv[1]); B = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
nl = int(sys.argv[4]) if len(sys.argv) > 4 else 1
base = gen.CONFIGS["long-video"]
wl = gen.DecodeWorkload(**{**base.__dict__, "name": "x", "B": B, "nv": nv, "k": max(1, nv // 10), "seq_lens": None})
xs = [gen.make_decode_inputs(wl, seed=100 + i, device="cuda") for i in range(nl)]
ws = svl.Workspace()
ws.get(svl.fresh_decode_workspace_size(wl.B, wl.H, wl.Hkv, wl.d, wl.k, wl.nv, wl.capacity))
for r in range(reps):
    for x in xs:
        out = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws)
    if os.environ.get("SYNC_EACH"):
        torch.cuda.synchronize()
torch.cuda.synchronize()
print("ok", B, nv, reps, nl)
