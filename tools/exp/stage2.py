import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
for name, n_q in (("long-video", 1), ("long-video", 32), ("long-video", 512), ("sweep", 1), ("multi-turn", 1)):
    base = gen.CONFIGS[name]
    wl = gen.DecodeWorkload(**{**base.__dict__, "n_q": n_q, "seq_lens": None})
    x = gen.make_decode_inputs(wl, seed=21, device="cuda")
    ws = svl.Workspace()
    ws.get(svl.retrieve_workspace_size(wl.B, n_q, wl.H, wl.Hkv, wl.d, wl.nv))
    ws.reset_flags()
    svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws)
    print(name, n_q, "generic path" if ws.flags() & 0x100 else "fast path", hex(ws.flags()))
    del x
