"""A/B timing of svl_question_attention (f1 attention output) vs flash_attn (library FA2)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2510_17777_b200 import svl, inputs as gen

def timeit(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    ts = []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(iters):
        flush.zero_()
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]

for n_q in (32, 128, 512):
    wl = gen.DecodeWorkload("lv", 1, 28, 4, 128, 32, 32768, 480 + 256, 3277, n_q, 256)
    x = gen.make_decode_inputs(wl, seed=1, device="cuda")
    L = int(x["seq_len"][0])
    out, lse = svl.question_attention(x["q"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv)
    t_full = timeit(lambda: svl.question_attention(x["q"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, out=out))
    t_lse = timeit(lambda: svl.question_attention(x["q"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, lse_in=lse, out=out))
    flops = 4.0 * wl.H * n_q * L * wl.d
    line = f"n_q={n_q} L={L}: svl {t_full:.1f} us (lse_in {t_lse:.1f} us, {flops / t_lse / 1e6:.0f} TFLOP/s)"
    try:
        from flash_attn import flash_attn_func
        q = x["q"]                                        # [B][n_q][H][d]
        k = x["K"][:, :, :L].transpose(1, 2).contiguous()  # [B][L][Hkv][d]
        v = x["V"][:, :, :L].transpose(1, 2).contiguous()
        o2 = flash_attn_func(q, k, v, causal=True)
        t_fa = timeit(lambda: flash_attn_func(q, k, v, causal=True))
        err = (o2.float() - out).abs().max().item()
        line += f"; flash_attn {t_fa:.1f} us (max |diff| {err:.2e})"
    except Exception as e:
        line += f"; flash_attn unavailable ({type(e).__name__}: {e})"
    print(line, flush=True)
