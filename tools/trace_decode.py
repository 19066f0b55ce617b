"""Phase timeline of the split decode kernel (SVL_TRACE=1 stamps), cold L2 (28 rotating layers).
usage: python tools/trace_decode.py [config]"""
import os, sys
os.environ["SVL_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
name = sys.argv[1] if len(sys.argv) > 1 else "long-video"
wl = gen.CONFIGS[name]
NL = 28
xs = [gen.make_decode_inputs(wl, seed=s, device="cuda") for s in range(NL)]
idx = [svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k).clone() for x in xs]
ws = svl.Workspace()
ws.get(svl.sparse_decode_workspace_size(wl.B, wl.H, wl.Hkv, wl.d, wl.k, wl.nv, wl.capacity))
for rep in range(2):
    for i in range(NL):
        x = xs[i]
        if i == NL - 1:
            ws.buf[256:256 + (1 << 20)].zero_()
        svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx[i], ws=ws)
torch.cuda.synchronize()
tr = ws.buf[256:256 + (1 << 20)].view(torch.int64)[: 4096 * 16].view(-1, 16).cpu()
tr = tr[tr[:, 0] > 0]
t0 = tr[:, 0].min()
names = {0: "start", 1: "batch0 ready", 2: "batch1 ready", 3: "batch2 ready", 10: "compute done", 11: "partial",
         12: "cl.sync", 13: "merge", 14: "end"}
print(f"{name} decode: {tr.shape[0]} CTAs (us from first start: min / median / max)")
for ph, nm in names.items():
    col = tr[:, ph]
    if (col == 0).any():
        continue
    v = (col - t0).double() / 1e3
    print(f"  {ph:2d} {nm:14s} {v.min():8.2f} {v.median():8.2f} {v.max():8.2f}")
