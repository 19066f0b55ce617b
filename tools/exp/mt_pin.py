"""multi-turn fresh step: planner choice vs the fused kernel pinned to 8 / 16 CTAs per unit."""
import sys, torch
sys.path.insert(0, ".")
from paper_2510_17777_b200 import svl, inputs as gen
wl = gen.CONFIGS["multi-turn"]
nl = 8
xs = [gen.make_decode_inputs(wl, seed=s, device="cuda") for s in range(nl)]
for name, flags in (("planner", 0), ("fused-8", svl.SVL_PIN_SPLITS(8)), ("fused-16", svl.SVL_PIN_SPLITS(16))):
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
    for _ in range(5): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(50): g.replay()
    e1.record(); torch.cuda.synchronize()
    print(name, f"{e0.elapsed_time(e1) * 1e3 / 50 / nl:.2f} us/layer", flush=True)
