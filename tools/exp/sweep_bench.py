"""Fresh-retrieval decode step on the BASELINE throughput-sweep config (B = 16, 64k visual,
k = 10 %): per-layer time of svl_fresh_decode_step (two-call path at 64k per unit) over
rotating layers, as d5 bytes / time.  usage: python tools/exp/sweep_bench.py [layers]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
wl = gen.CONFIGS["sweep"]
NL = int(sys.argv[1]) if len(sys.argv) > 1 else 3
xs = [gen.make_decode_inputs(wl, seed=300 + i, device="cuda") for i in range(NL)]
ws = svl.Workspace()
ws.get(svl.fresh_decode_workspace_size(wl.B, wl.H, wl.Hkv, wl.d, wl.k, wl.nv, wl.capacity))
idx = torch.empty(wl.B, wl.Hkv, wl.k, dtype=torch.int32, device="cuda")
out = torch.empty(wl.B, wl.H, wl.d, device="cuda")
def step():
    for x in xs:
        svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, idx_out=idx, out=out, ws=ws)
step(); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        step()
for _ in range(3): g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): g.replay()
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 10 / NL
T = wl.vb + wl.t_after
row = wl.d * 2
nbytes = wl.B * wl.Hkv * (wl.nv * row + wl.k * 2 * row + T * 2 * row) + wl.B * wl.H * wl.d * 6 + wl.B * wl.Hkv * wl.k * 4
print(f"sweep B={wl.B} nv={wl.nv} k={wl.k}: {us:.1f} us/layer, {nbytes / us / 1e3:.0f} GB/s ({nbytes/1e6:.1f} MB/layer)")
