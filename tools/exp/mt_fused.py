"""Fresh step on multi-turn (B = 8, 16k) and long-video B = 2/4: planner vs pinned fused (multi-wave)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
_a = torch.empty(1 << 28, dtype=torch.uint8, device="cuda"); _b = torch.empty_like(_a)
for _ in range(1000): _b.copy_(_a)
def run(wl, nl, flags):
    xs = [gen.make_decode_inputs(wl, seed=s, device="cuda") for s in range(nl)]
    ws = svl.Workspace()
    outs = [torch.empty(wl.B, wl.H, wl.d, device="cuda") for _ in range(nl)]
    idxs = [torch.empty(wl.B, wl.Hkv, wl.k, dtype=torch.int32, device="cuda") for _ in range(nl)]
    def body():
        for l in range(nl):
            x = xs[l]
            svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, out=outs[l],
                                  idx_out=idxs[l], ws=ws, flags=flags)
    body(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            body()
    for _ in range(10): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100): g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / 100 / nl
base = gen.CONFIGS["long-video"]
def mk(B, nv):
    return gen.DecodeWorkload(**{**base.__dict__, "name": f"b{B}n{nv}", "B": B, "nv": nv, "k": nv // 10, "seq_lens": None})
for name, wl, nl in [("lv B3", mk(3, 32768), 10), ("lv B4", mk(4, 32768), 7), ("24k B4", mk(4, 24576), 9),
                     ("16k B4", mk(4, 16384), 14), ("16k B6", mk(6, 16384), 10), ("32k B5", mk(5, 32768), 6)]:
    res = {}
    for tag, fl in [("planner", 0), ("fused16", svl.SVL_PIN_SPLITS(16)), ("unfused", svl.SVL_FRESH_UNFUSED)]:
        try:
            res[tag] = round(run(wl, nl, fl), 2)
        except Exception as e:
            res[tag] = str(e)[:40]
    print(name, res)
