"""Round-2 additions under compute-sanitizer: svl_question_attention (tcgen05 output pass) and
svl_retrieve past one wave of clusters (relevance pass + refined mode-3 select).
python tools/exp/sanitize_new.py N  (N calls each, compared bitwise with the first)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wq = gen.DecodeWorkload("qa", 1, 28, 4, 128, 32, 1500, 333, 64, 16, 256)
xq = gen.make_decode_inputs(wq, seed=3, device="cuda")
wr = gen.DecodeWorkload("many", 10, 28, 4, 128, 32, 16384, 300, 1638, 1, 256)
xr = gen.make_decode_inputs(wr, seed=4, device="cuda")
ws = svl.Workspace()
o0, l0 = svl.question_attention(xq["q"], xq["K"], xq["V"], xq["seq_len"], wq.vb, wq.nv, ws=ws)
o0, l0 = o0.clone(), l0.clone()
r0 = svl.retrieve(xr["q"], xr["K"], xr["seq_len"], wr.vb, wr.nv, wr.k, ws=ws).clone()
bad = 0
for _ in range(N):
    o, l = svl.question_attention(xq["q"], xq["K"], xq["V"], xq["seq_len"], wq.vb, wq.nv, ws=ws)
    r = svl.retrieve(xr["q"], xr["K"], xr["seq_len"], wr.vb, wr.nv, wr.k, ws=ws)
    bad += int(not (torch.equal(o, o0) and torch.equal(l, l0) and torch.equal(r, r0)))
torch.cuda.synchronize()
print(f"question attention + many-unit retrieve: {N} calls, {bad} differ from the first; device flags {ws.flags()}")
