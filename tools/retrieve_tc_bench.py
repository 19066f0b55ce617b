"""Time the tensor-core retrieve (svl_retrieve, n_q * g > 32) on the long-video cache.
usage: python tools/retrieve_tc_bench.py [n_q ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl

base = gen.CONFIGS["long-video"]
for n_q in [int(a) for a in sys.argv[1:]] or [32, 128, 512]:
    wl = gen.DecodeWorkload(**{**base.__dict__, "name": f"q{n_q}", "n_q": n_q, "seq_lens": None})
    x = gen.make_decode_inputs(wl, seed=21, device="cuda")
    ws = svl.Workspace()
    idx = torch.empty(wl.B, wl.Hkv, wl.k, dtype=torch.int32, device="cuda")
    lse = torch.zeros(wl.B, n_q, wl.H, dtype=torch.float32, device="cuda") + 9.0
    for name, kw in (("full", {}), ("lse_in", {"lse_in": lse})):
        f = lambda: svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, idx_out=idx, ws=ws, **kw)
        f(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                f()
        for _ in range(3): g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): g.replay()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        L, units = wl.seq_len, wl.B * wl.Hkv
        p0 = wl.g * (n_q * (L - n_q) + n_q * (n_q + 1) // 2)
        fl = 2 * wl.d * units * ((p0 if name == "full" else 0) + n_q * wl.g * wl.nv)
        print(f"n_q={n_q:4d} rows/unit={n_q * wl.g:5d} {name:7s}: {us:9.1f} us  {fl / us / 1e6:7.1f} TFLOP/s")
