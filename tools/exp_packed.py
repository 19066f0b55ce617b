"""Steady decode: gathered (svl_sparse_decode_attn with indices) vs packed
contiguous KV (the same rows copied once, attended as a dense span) -- f2 probe.
28 rotating layers in one CUDA graph."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl

wl = gen.CONFIGS["long-video"]
NL = 28
L = []
for l in range(NL):
    x = gen.make_decode_inputs(wl, seed=200 + l, device="cuda")
    idx = svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k).clone()
    rows = torch.cat([torch.arange(wl.vb, device="cuda"),
                      wl.vb + idx[0, 0].long()], 0)  # per-head rows differ: build per head
    Kp = torch.empty(wl.B, wl.Hkv, wl.vb + wl.k + (wl.seq_len - wl.vb - wl.nv), wl.d, dtype=torch.bfloat16, device="cuda")
    Vp = torch.empty_like(Kp)
    for G in range(wl.Hkv):
        r = torch.cat([torch.arange(wl.vb, device="cuda"), wl.vb + idx[0, G].long(),
                       torch.arange(wl.vb + wl.nv, wl.seq_len, device="cuda")])
        Kp[0, G] = x["K"][0, G, r]
        Vp[0, G] = x["V"][0, G, r]
    sl = torch.full((1,), Kp.shape[2], dtype=torch.int32, device="cuda")
    L.append((x, idx, Kp, Vp, sl))
ws = svl.Workspace()
outs = torch.empty(wl.B, wl.H, wl.d, device="cuda")


def gathered():
    for x, idx, Kp, Vp, sl in L:
        svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx, out=outs, ws=ws)


def packed():
    for x, idx, Kp, Vp, sl in L:
        svl.sparse_decode_attn(x["q_dec"], Kp, Vp, sl, 0, 0, None, out=outs, ws=ws)


def timeit(fn, reps=50):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps / NL


print(f"gathered {timeit(gathered):.2f} us/layer   packed {timeit(packed):.2f} us/layer")
