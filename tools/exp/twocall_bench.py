"""Two-call path timing per config: score / select / decode graphs (us per layer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
tag = sys.argv[1] if len(sys.argv) > 1 else ""
_a = torch.empty(1 << 28, dtype=torch.uint8, device="cuda"); _b = torch.empty_like(_a)
for _ in range(1000): _b.copy_(_a)
def timed(fn, n=30):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st): fn()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n
for name, nl in (("sweep", 3), ("multi-turn", 8), ("long-video", 8)):
    wl = gen.CONFIGS[name]
    xs = [gen.make_decode_inputs(wl, seed=s, device="cuda") for s in range(nl)]
    ws = svl.Workspace(); wsd = svl.Workspace()
    idx = [torch.empty(wl.B, wl.Hkv, wl.k, dtype=torch.int32, device="cuda") for _ in range(nl)]
    outs = [torch.empty(wl.B, wl.H, wl.d, device="cuda") for _ in range(nl)]
    sc = timed(lambda: [svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, flags=svl.SVL_RETRIEVE_SCORE_ONLY, idx_out=i, ws=ws) for x, i in zip(xs, idx)]) / nl
    se = timed(lambda: [svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k, flags=svl.SVL_RETRIEVE_SELECT_ONLY, idx_out=i, ws=ws) for x, i in zip(xs, idx)]) / nl
    de = timed(lambda: [svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, i, out=o, ws=wsd) for x, i, o in zip(xs, idx, outs)]) / nl
    fr = timed(lambda: [svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, idx_out=i, out=o, ws=ws) for x, i, o in zip(xs, idx, outs)]) / nl
    print(tag, name, f"score {sc:.1f} select {se:.1f} decode {de:.1f} fresh {fr:.1f} us/layer")
    del xs
