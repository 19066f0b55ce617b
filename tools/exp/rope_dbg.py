import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle
from paper_2510_17777_b200 import svl
oracle.build()
B, Hkv, d, vb, nv, ta, k, base = 1, 1, 128, 32, 4096, 300, 1024, float(sys.argv[1])
g = torch.Generator().manual_seed(5)
cap = vb + nv + ta + 7
K = torch.randn(B, Hkv, cap, d, generator=g).to(torch.bfloat16)
kept = torch.sort(torch.randperm(nv, generator=g)[:k]).values.to(torch.int32)[None]
seq = torch.tensor([vb + nv + ta], dtype=torch.int32)
Ko, _, sn = svl.rope_remap(K.cuda(), None, seq.cuda(), vb, nv, kept.cuda(), base)
ref, rows = oracle.rope_remap(K, seq.numpy(), vb, nv, kept.numpy(), base, cap_out=Ko.shape[2])
n = int(sn[0]); got = Ko.cpu()[0, 0, :n].double().numpy(); ex = ref[0, 0, :n]
err = np.abs(got - ex)
ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ex), 2.0 ** -126))) - 7)
bad = np.argwhere(err > ulp)
print("base", base, "bad", len(bad), "max", err.max())
for w, c in bad[:8]:
    print(w, c, got[w, c], ex[w, c], "row", rows[0][w])
