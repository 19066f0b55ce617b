"""28-layer graph of svl_fresh_decode_step on long-video (and nvila-4k): us/layer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
tag = sys.argv[1] if len(sys.argv) > 1 else ""
_a = torch.empty(1 << 28, dtype=torch.uint8, device="cuda"); _b = torch.empty_like(_a)
for _ in range(1000): _b.copy_(_a)
for name, nl in [c for c in (("long-video", 28), ("nvila-4k", 77)) if c[0] in os.environ.get("CFGS", "long-video,nvila-4k")]:
    wl = gen.CONFIGS[name]
    xs = [gen.make_decode_inputs(wl, seed=s, device="cuda") for s in range(nl)]
    ws = svl.Workspace()
    outs = [torch.empty(wl.B, wl.H, wl.d, device="cuda") for _ in range(nl)]
    idxs = [torch.empty(wl.B, wl.Hkv, wl.k, dtype=torch.int32, device="cuda") for _ in range(nl)]
    def body():
        for l in range(nl):
            x = xs[l]
            svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, out=outs[l],
                                  idx_out=idxs[l], ws=ws)
    body(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            body()
    for _ in range(20): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(300): g.replay()
    e1.record(); torch.cuda.synchronize()
    print(tag, name, f"{e0.elapsed_time(e1) * 1e3 / 300 / nl:.2f} us/layer")
    del xs
