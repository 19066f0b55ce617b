"""N back-to-back calls of the fresh step, the steady decode and the two-call retrieve on a
config, each output compared bitwise with the first call (a debug SVL_DEBUG_TRAP build traps
on an out-of-range V slot or gathered row).  python tools/exp/many_calls.py config N"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
name, N = sys.argv[1], int(sys.argv[2])
wl = gen.CONFIGS[name]
x = gen.make_decode_inputs(wl, seed=99, device="cuda")
ws = svl.Workspace()
o0, i0 = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws)
o0, i0 = o0.clone(), i0.clone()
d0, _ = svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, i0, ws=ws)
d0 = d0.clone()
r0 = svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws).clone()
bad = 0
for it in range(N):
    o, i = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws)
    d, _ = svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, i0, ws=ws)
    r = svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws)
    # (i0 and the cache are not written by the retrieve before it: the early-gather path)
    ds, _ = svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, i0,
                                   flags=svl.SVL_DECODE_STATIC_PREFIX, ws=ws)
    if it % 100 == 99 or it == N - 1:
        torch.cuda.synchronize()
    bad += int(not (torch.equal(o, o0) and torch.equal(i, i0) and torch.equal(d, d0) and torch.equal(ds, d0) and torch.equal(r, r0)))
torch.cuda.synchronize()
print(f"{name}: {N} x (fresh step + steady decode + retrieve + early-gather decode): {bad} calls differ from the first; "
      f"device flags {ws.flags()}")
