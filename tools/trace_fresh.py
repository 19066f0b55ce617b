"""Phase timeline of the fused fresh-step kernel (SVL_TRACE=1 debug stamps).
usage: python tools/trace_fresh.py [config]"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if "SVL_LIB" not in os.environ:  # a phase-stamp build (SVL_TRACE_BUILD) in build/trace/
    env = dict(os.environ, SVL_VARIANT="trace", SVL_DEFS="-DSVL_TRACE_BUILD=1")
    subprocess.run([sys.executable, "-m", "paper_2510_17777_b200.build"], cwd=ROOT, env=env, check=True,
                   stdout=subprocess.DEVNULL)
    os.environ["SVL_LIB"] = os.path.join(ROOT, "build", "trace", "libsparsevila.so")
import torch
from paper_2510_17777_b200 import inputs as gen, svl
name = sys.argv[1] if len(sys.argv) > 1 else "long-video"
wl = gen.CONFIGS[name]
NL = int(os.environ.get("TRACE_LAYERS", "28"))  # rotating layers: the traced one is cold in L2
xs = [gen.make_decode_inputs(wl, seed=s, device="cuda") for s in range(NL)]
ws = svl.Workspace()
ws.get(max(svl.fresh_decode_workspace_size(wl.B, wl.H, wl.Hkv, wl.d, wl.k, wl.nv, wl.capacity), 1024 + (1 << 20)))
_a = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
_b = torch.empty_like(_a)
for _ in range(2000):  # ~1 s of copies: the SM clock ramps up from idle
    _b.copy_(_a)
for rep in range(2):
    for it in range(NL):
        x = xs[it]
        if it == NL - 1:
            ws.buf[1024:1024 + (1 << 20)].zero_()
        svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws)
torch.cuda.synchronize()
tr = ws.buf[1024:1024 + (1 << 20)].view(torch.int64)[: 2048 * 64].view(-1, 64).cpu()
tr = tr[tr[:, 0] > 0]
# slots 0 / 10: global timer (ns); 30 / 31: SM cycles at those points; every other slot: SM
# cycles -> ns on the global timeline at the CTA's measured clock
ratio = (tr[:, 10] - tr[:, 0]).double() / (tr[:, 31] - tr[:, 30]).double()
conv = tr.clone()
for j in range(64):
    if j in (0, 10, 30, 31):
        continue
    nz = tr[:, j] != 0
    # (int64 offset first: ~1.8e18 ns does not survive a double addition below 256 ns)
    conv[nz, j] = tr[nz, 0] + ((tr[nz, j] - tr[nz, 30]).double() * ratio[nz]).round().long()
cyc_ratio = ratio
tr, raw = conv, tr
t0 = tr[:, 0].min()
names = {0: "start", 1: "stream+textV", 2: "lse", 3: "hist+thr", 4: "select", 5: "Ptab+Vwait", 6: "PV", 7: "O+l",
         8: "merge-sync", 9: "merge", 10: "end", 11: "assign+push", 12: "gather-issue"}
print(f"{name}: {tr.shape[0]} CTAs; phase end times (us, min/median/max over CTAs, from first start)")
for ph, nm in names.items():
    col = tr[:, ph]
    if (col == 0).any():
        continue
    v = (col - t0).double() / 1e3
    print(f"  {ph:2d} {nm:10s} {v.min():8.2f} {v.median():8.2f} {v.max():8.2f}")

post = {13: "LSE warps: last stage", 14: "LSE warps: folded", 15: "LDS warps: folded", 29: "MMA warp: done"}
print("end of the stream (us from start, median):")
for j, nm in post.items():
    col = tr[:, j]
    if (col == 0).any():
        continue
    print(f"   {nm:24s} {((col - tr[:, 0]).double() / 1e3).median().item():8.2f}")

lean = {26: "keys done", 27: "B1", 28: "w0: hists landed", 12: "U: B3+slots", 11: "U: V issued", 16: "D: V landed", 17: "D: PV above", 18: "D: cut recv", 19: "D: PV cands",
        20: "S: cands landed", 21: "S: cut", 22: "S: emitted", 6: "final sync", 23: "lred/octa",
        24: "sync", 25: "lh", 56: "U1 (counts) + B3", 57: "U TMEM loads", 58: "U slots/P/push", 59: "U gathers",
        60: "U text P + pads"}
print("split pipeline (us from the threshold stamp, median / max over CTAs):")
for j, nm in lean.items():
    col = tr[:, j]
    if (col == 0).any():
        continue
    v = (col - tr[:, 3]).double() / 1e3
    print(f"   {nm:22s} {v.median().item():8.2f} {v.max().item():8.2f}")
sub = ["cand-hist", "find", "flags", "mine", "scan", "off", "-", "-", "-", "-", "-", "-", "-"]
print("resolve internals (us from gather-issue, median):")
for j, nm in (enumerate(sub) if not (tr[:, 12] == 0).any() and (tr[:, 11] > tr[:, 12]).all() else []):
    col = tr[:, 16 + j]
    if (col == 0).any():
        continue
    print(f"   {nm:10s} {((col - tr[:, 12]).double() / 1e3).median().item():8.2f}")

hsub = {8: "keys+hist", 9: "hist-sync", 10: "fold+push", 11: "cl.sync", 12: "sum+find"}
print("histogram internals (us from lse stamp, median):")
for j, nm in hsub.items():
    col = tr[:, 16 + j]
    if (col == 0).any():
        continue
    print(f"   {nm:10s} {((col - tr[:, 2]).double() / 1e3).median().item():8.2f}")

print("stage arrivals (us from start, median):", " ".join(
    f"{((tr[:, 32 + i] - tr[:, 0]).double() / 1e3).median().item():.2f}" for i in range(24) if not (tr[:, 32 + i] == 0).any()))

cyc = (raw[:, 31] - raw[:, 30]).double()
ns = (raw[:, 10] - raw[:, 0]).double()
print(f"SM clock during the kernel (clock64 / globaltimer, median over CTAs): {(cyc / ns).median().item() * 1e3:.0f} MHz")

print("LDS-warp stage done (us from start, median):", " ".join(
    f"{((tr[:, 48 + i] - tr[:, 0]).double() / 1e3).median().item():.2f}" for i in range(8) if not (tr[:, 48 + i] == 0).any()))
