"""Which selection path runs?  Needs a build with -DSVL_EXP_FLAG_STAGE2 (device flags
0x100 = generic radix fallback, 0x200 = the cut-bin refinement round ran)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2510_17777_b200 import svl, inputs as gen
cases = dict(gen.CONFIGS)
cases["smooth-64k"] = gen.DecodeWorkload("smooth", 1, 28, 4, 128, 32, 65536, 300, 6554, 1, 65536, 0, 0)
cases["smooth-32k"] = gen.DecodeWorkload("smooth", 1, 28, 4, 128, 32, 32768, 300, 3277, 1, 32768, 0, 0)
for name, wl in cases.items():
    x = gen.make_decode_inputs(wl, seed=1, device="cuda")
    ws = svl.Workspace()
    svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws)
    torch.cuda.synchronize()
    f1 = ws.flags()
    ws2 = svl.Workspace()
    svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws2)
    torch.cuda.synchronize()
    print(name, "retrieve flags", hex(f1), "fresh flags", hex(ws2.flags()),
          "fused" if svl.fresh_uses_fused(wl.B, wl.H, wl.Hkv, wl.d, wl.nv, wl.capacity) else "two-call", flush=True)
