"""Time svl_fresh_decode_step on a custom long-video-shaped workload
(28 rotating layers in one CUDA graph, like bench.py) -- design experiments.
usage: SVL_LIB=build/<variant>/libsparsevila.so python tools/exp_fused.py NV [B] [REPS]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl

nv = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
base = gen.CONFIGS["long-video"]
wl = gen.DecodeWorkload(**{**base.__dict__, "name": f"lv{nv}", "B": B, "nv": nv, "k": max(1, nv // 10),
                           "seq_lens": None})
NL = 28
layers = [gen.make_decode_inputs(wl, seed=100 + i, device="cuda") for i in range(NL)]
ws = svl.Workspace()
ws.get(svl.fresh_decode_workspace_size(wl.B, wl.H, wl.Hkv, wl.d, wl.k, wl.nv, wl.capacity))
outs = []


def step():
    for x in layers:
        svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, ws=ws)


step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        step()
torch.cuda.synchronize()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps / NL
kbytes = wl.B * wl.Hkv * (wl.nv + wl.seq_len - wl.vb - wl.nv + wl.vb) * wl.d * 2
print(f"{os.environ.get('SVL_LIB', 'default')}: nv={nv} B={B}: {us:.2f} us/layer; K stream {kbytes / us / 1e3:.0f} GB/s-equivalent")
