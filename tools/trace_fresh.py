"""Phase timeline of the fused fresh-step kernel (SVL_TRACE=1 debug stamps)."""
import os, sys
os.environ["SVL_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
name = sys.argv[1] if len(sys.argv) > 1 else "long-video"
wl = gen.CONFIGS[name]
xs = [gen.make_decode_inputs(wl, seed=s, device="cuda") for s in range(6)]
ws = svl.Workspace()
ws.get(svl.fresh_decode_workspace_size(wl.B, wl.H, wl.Hkv, wl.d, wl.k, wl.nv, wl.capacity))
for it in range(6):
    x = xs[it]
    ws.buf[256:256 + (1 << 20)].zero_()
    torch.cuda.synchronize()
    svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws)
    torch.cuda.synchronize()
tr = ws.buf[256:256 + (1 << 20)].view(torch.int64)[: 2048 * 32].view(-1, 32).cpu()
tr = tr[tr[:, 0] > 0]
t0 = tr[:, 0].min()
names = ["start", "stream", "lse", "keys", "topk", "emit+M", "V+PV", "Ored", "merge-sync", "merge", "end", "keys#1"]
print(f"{name}: {tr.shape[0]} CTAs; phase end times (us, min/median/max over CTAs, from first start)")
for ph in range(12):
    v = (tr[:, ph] - t0).double() / 1e3
    print(f"  {ph:2d} {names[ph]:10s} {v.min():8.2f} {v.median():8.2f} {v.max():8.2f}")
cyc = (tr[:, 13] - tr[:, 12]).double()
ns = (tr[:, 3] - tr[:, 2]).double()
print("keys phase: cycles median", cyc.median().item(), "ns median", ns.median().item(), "=> GHz", (cyc / ns).median().item())

tn = ["push1", "sync1", "find1", "state1", "candpush+sync", "kth", "flags", "end"]
print("topk internals (us from keys end, median over CTAs):")
for j, nm in enumerate(tn):
    v = (tr[:, 16 + j] - tr[:, 3]).double() / 1e3
    print(f"   {nm:14s} {v.median().item():8.2f}")
