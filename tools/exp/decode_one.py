"""A few steady-decode calls on one config (for ncu): python tools/exp/decode_one.py [config] [calls]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
name = sys.argv[1] if len(sys.argv) > 1 else "long-video"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 8
wl = gen.CONFIGS[name]
xs = [gen.make_decode_inputs(wl, seed=s, device="cuda") for s in range(4)]
idx = [svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k).clone() for x in xs]
ws = svl.Workspace()
for i in range(calls):
    x = xs[i % 4]
    svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx[i % 4], ws=ws)
torch.cuda.synchronize()
