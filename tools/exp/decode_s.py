import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
wl = gen.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "sweep"]
xs = [gen.make_decode_inputs(wl, seed=300 + i, device="cuda") for i in range(2)]
idx = [torch.sort(torch.randperm(wl.nv, device="cuda")[:wl.k]).values.to(torch.int32).expand(wl.B, wl.Hkv, wl.k).contiguous() for _ in xs]
out = torch.empty(wl.B, wl.H, wl.d, device="cuda")
ws = svl.Workspace()
f = lambda: [svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, i, out=out, ws=ws) for x, i in zip(xs, idx)]
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
us = e0.elapsed_time(e1) * 1e3 / 20 / len(xs)
T = wl.vb + wl.t_after
nb = wl.B * wl.Hkv * (wl.k + T) * 2 * wl.d * 2
print(f"{os.environ.get('SVL_DECODE_S', 'plan')}: {us:.1f} us/layer {nb / us / 1e3:.0f} GB/s")
