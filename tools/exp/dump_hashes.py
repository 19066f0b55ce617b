"""Hash svl_fresh_decode_step outputs over configs x seeds (compare two builds bitwise).
usage: SVL_LIB=... python tools/exp/dump_hashes.py out.txt"""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_17777_b200 import inputs as gen, svl
cfgs = dict(gen.CONFIGS)
base = gen.CONFIGS["long-video"]
cfgs["lv-b8"] = gen.DecodeWorkload(**{**base.__dict__, "name": "lvb8", "B": 8, "seq_lens": None})
lines = []
for name in ["toy", "nvila-4k", "long-video", "multi-turn", "lv-b8"]:
    wl = cfgs[name]
    for seed in range(6):
        x = gen.make_decode_inputs(wl, seed=seed, device="cuda")
        for rep in range(2):
            out, idx = svl.fresh_decode_step(x["q_dec"], x["K"], x["V"], x["seq_len"], wl.vb, wl.nv, wl.k)
            torch.cuda.synchronize()
            h = hashlib.sha1(out.cpu().numpy().tobytes() + idx.cpu().numpy().tobytes()).hexdigest()[:16]
            lines.append(f"{name} {seed} {rep} {h}")
open(sys.argv[1], "w").write("\n".join(lines) + "\n")
print("done", len(lines))
