"""How often does SVL_DECODE_STATIC_PREFIX's seq_len speculation miss when the upstream PDL
kernel overwrites the decode's seq_len words?  (needs a build with -DSVL_EXP_MISS_FLAG=1:
a miss raises device flag bit 16).  UP=fresh|decode picks the upstream writer; the sequence
[reset seq_len, upstream, decode] is replayed from a CUDA graph (eager launches leave CPU gaps
between the kernels, so nothing races)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
up = os.environ.get("UP", "fresh")
for name in ("toy", "nvila-4k", "long-video"):
    wl = gen.CONFIGS[name]
    x = gen.make_decode_inputs(wl, seed=95, device="cuda")
    idx = svl.retrieve(x["q"], x["K"], x["seq_len"], wl.vb, wl.nv, wl.k).clone()
    buf = torch.zeros(wl.B, wl.H, wl.d, device="cuda")
    seq_view = buf.view(-1).view(torch.int32)[:wl.B]
    ws_f, ws_d = svl.Workspace(), svl.Workspace()
    a = torch.empty(wl.B, wl.H, wl.d, device="cuda")

    def body():
        seq_view.copy_(x["seq_len"])
        if up == "decode":
            svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, idx, out=buf, ws=ws_f)
        else:
            svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k, out=buf, ws=ws_f)
        svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], seq_view, wl.vb, wl.nv, idx,
                               flags=svl.SVL_DECODE_STATIC_PREFIX, out=a, ws=ws_d)
    body(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            body()
    miss, bad = 0, 0
    for it in range(50):
        ws_d.reset_flags()
        g.replay()
        torch.cuda.synchronize()
        miss += int(bool(ws_d.flags() & 16))
        ref, _ = svl.sparse_decode_attn(x["q_dec"], x["K"], x["V"], seq_view, wl.vb, wl.nv, idx)
        bad += int(not torch.equal(a, ref))
    print(name, up, "speculation misses:", miss, "/ 50; results differing from the plain call:", bad)
