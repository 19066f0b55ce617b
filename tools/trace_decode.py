"""Phase timeline of the steady decode kernel (svl_sparse_decode_attn), from
globaltimer stamps of a SVL_TRACE_BUILD library (built here as build/trace/),
cold L2 (28 rotating layers, the last one traced).
usage: python tools/trace_decode.py [config] [pin]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if "SVL_LIB" not in os.environ:
    env = dict(os.environ, SVL_VARIANT="trace", SVL_DEFS="-DSVL_TRACE_BUILD=1")
    subprocess.run([sys.executable, "-m", "paper_2510_17777_b200.build"], cwd=ROOT, env=env, check=True,
                   stdout=subprocess.DEVNULL)
    os.environ["SVL_LIB"] = os.path.join(ROOT, "build", "trace", "libsparsevila.so")
import torch  # noqa: E402

from paper_2510_17777_b200 import inputs as gen, svl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "long-video"
pin = int(sys.argv[2]) if len(sys.argv) > 2 else 0
flags = (svl.SVL_PIN_SPLITS(pin) if pin else 0) | int(os.environ.get("DFLAGS", "0"), 0)
wl = gen.CONFIGS[name]
NL = 28 if wl.B * wl.nv <= 65536 else 3
xs = [gen.make_decode_inputs(wl, seed=s, device="cuda") for s in range(NL)]
idx = [svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k).clone() for x in xs]
base = svl.sparse_decode_workspace_size(wl.B, wl.H, wl.Hkv, wl.d, wl.k, wl.nv, wl.capacity, flags)
ws = svl.Workspace()
ws.get(base + (1 << 20))
tr_view = ws.buf[ws.buf.numel() - (1 << 20):]
# ~1 s of back-to-back copies first: the SM clock ramps up from idle under load
# (a copy, not a GEMM: a power-capped GEMM leaves the clock low)
a = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
b = torch.empty_like(a)
for _ in range(2000):
    b.copy_(a)
for rep in range(3):
    for i in range(NL):
        x = xs[i]
        if rep == 2 and i == NL - 1:
            tr_view.zero_()
        svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx[i], flags=flags, ws=ws)
torch.cuda.synchronize()
tr = tr_view.view(torch.int64)[: 4096 * 16].view(-1, 16).cpu()
tr = tr[tr[:, 0] > 0]
# stamps 0..13: SM cycles (clock64) of the CTA; 14 / 15: globaltimer at start / end
f_ghz = ((tr[:, 7] - tr[:, 0]).double() / (tr[:, 15] - tr[:, 14]).double())
print(f"SM clock during the kernel (clock64 / globaltimer, median over CTAs): {f_ghz.median() * 1e3:.0f} MHz")
names = {6: "PDL wait released", 1: "seq_len read", 2: "row ids", 3: "batch0 landed", 4: "compute done",
         10: "O staged (cross-warp)", 11: "CTA M / l", 12: "cluster_wait",
         5: "partial stored/pushed", 8: "partials landed", 9: "merged", 7: "end"}
print(f"{name} decode pin={pin}: {tr.shape[0]} CTAs; per-CTA cycles from its start -> us at its clock "
      f"(min / median / max); kernel span {((tr[:, 15].max() - tr[:, 14].min()) / 1e3).item():.2f} us")
for ph, nm in names.items():
    ok = tr[:, ph] > 0
    if not ok.any():
        continue
    v = (tr[ok, ph] - tr[ok, 0]).double() / f_ghz[ok] / 1e3
    print(f"  {ph:2d} {nm:22s} {v.min():8.2f} {v.median():8.2f} {v.max():8.2f}")
# the same phases from the CTA's own PDL release (stamp 6): the critical path after the wait
ok6 = tr[:, 6] > 0
if ok6.any():
    print("  from the PDL release (min / median / max):")
    for ph, nm in names.items():
        ok = ok6 & (tr[:, ph] > 0)
        if ph == 6 or not ok.any():
            continue
        v = (tr[ok, ph] - tr[ok, 6]).double() / f_ghz[ok] / 1e3
        print(f"  {ph:2d} {nm:22s} {v.min():8.2f} {v.median():8.2f} {v.max():8.2f}")
