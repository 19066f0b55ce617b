"""Steady-decode timing sweep: 28-layer CUDA graph of svl_sparse_decode_attn per config and
pinned split count (0 = planner).  python tools/exp/decode_bench.py [lib tag]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
import bench

def run(name, pins, layers=28, steps=200):
    if name.startswith("lvB"):  # long-video at batch B (e.g. lvB2)
        base = gen.CONFIGS["long-video"]
        wl = gen.DecodeWorkload(**{**base.__dict__, "name": name, "B": int(name[3:]), "seq_lens": None})
    else:
        wl = gen.CONFIGS[name]
    nl = layers if name != "sweep" else 3
    xs = [gen.make_decode_inputs(wl, seed=500 + l, device="cuda") for l in range(nl)]
    idx = [torch.sort(torch.stack([torch.stack([torch.randperm(wl.nv, device="cuda")[:wl.k] for _ in range(wl.Hkv)])
                                   for _ in range(wl.B)]), -1)[0].to(torch.int32).contiguous() for _ in range(nl)]
    outs = [torch.empty(wl.B, wl.H, wl.d, device="cuda") for _ in range(nl)]
    res = {}
    for pin in pins:
        ws = svl.Workspace()
        fl = (svl.SVL_PIN_SPLITS(abs(pin)) if pin else 0) | (svl.SVL_DECODE_GRID_MERGE if pin < 0 else 0)
        fl |= svl.SVL_DECODE_STATIC_PREFIX if os.environ.get("DSTATIC") == "1" else 0
        def body():
            for l in range(nl):
                svl.sparse_decode_attn(xs[l]["q_dec"], xs[l]["K"], xs[l]["V"], xs[l]["seq_len"], wl.vb, wl.nv,
                                       idx[l], flags=fl, out=outs[l], ws=ws)
        try:
            body(); torch.cuda.synchronize()
        except Exception as e:
            res[pin] = str(e)[:60]; continue
        g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                body()
        for _ in range(10): g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps): g.replay()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / steps / nl
        res[pin] = round(us, 2)
        # single cold layer: events around one launch after an L2 flush
        flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
        ts = []
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); svl.sparse_decode_attn(xs[0]["q_dec"], xs[0]["K"], xs[0]["V"], xs[0]["seq_len"], wl.vb, wl.nv,
                                               idx[0], flags=fl, out=outs[0], ws=ws); b.record()
            torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
        res[f"{pin}_cold"] = round(sorted(ts)[len(ts) // 2], 2)
    nb = bench.step_bytes(wl)["decode"]
    print(json.dumps({"config": name, "bytes": nb, "us": res,
                      "GBs": {k: round(nb / (v * 1e-6) / 1e9) for k, v in res.items() if isinstance(v, float)}}))

tag = sys.argv[1] if len(sys.argv) > 1 else ""
_a = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
_b = torch.empty_like(_a)
for _ in range(2000):  # ~1 s of copies: the SM clock ramps up from idle (a GEMM would power-cap it)
    _b.copy_(_a)
torch.cuda.synchronize()
print("lib", svl.LIB_PATH, tag)
_cf = os.environ.get("DCFGS")
if _cf is None:
    run("long-video", [0, 16, -16, 8, 4])
    run("nvila-4k", [0, 16, 8])
    run("multi-turn", [0, -4, 4, 2])
    run("sweep", [0, -2, 2, 1])
else:  # e.g. DCFGS="long-video:0,16;nvila-4k:0"
    for item in _cf.split(";"):
        nm, pins = item.split(":")
        run(nm, [int(v) for v in pins.split(",")])
