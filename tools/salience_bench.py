import os, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2510_17777_b200 import inputs as gen, svl
pw = gen.PrefillWorkload()
px = gen.make_prefill_inputs(pw, seed=7, device="cuda")
sal = torch.empty(pw.F, pw.Nf, dtype=torch.float32, device="cuda")
ws = svl.Workspace()
for _ in range(3): svl.salience(px["Qe"], px["Ke"], 0, 2, out=sal, ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): svl.salience(px["Qe"], px["Ke"], 0, 2, out=sal, ws=ws)
e1.record(); torch.cuda.synchronize()
print(os.environ.get("SVL_LIB", "default"), "salience ms", e0.elapsed_time(e1) / 20)
