"""svl_question_attention on the long-video cache, n_q = 128, lse_in given (for ncu)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2510_17777_b200 import svl, inputs as gen
wl = gen.DecodeWorkload("lv", 1, 28, 4, 128, 32, 32768, 480 + 256, 3277, 128, 256)
x = gen.make_decode_inputs(wl, seed=1, device="cuda")
out, lse = svl.question_attention(x["q"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv)
for _ in range(2):
    svl.question_attention(x["q"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, lse_in=lse, out=out)
torch.cuda.synchronize()
print("ok")
