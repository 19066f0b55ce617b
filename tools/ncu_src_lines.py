"""Top CUDA source lines by warp-stall samples from
`ncu -i X.ncu-rep --page source --csv --print-source sass,cuda`.
usage: python tools/ncu_src_lines.py file.csv [N]"""
import csv, io, sys

path = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows, cur = [], None
for blk in open(path).read().split('"File Path",')[1:]:
    lines = blk.splitlines()
    fname = lines[0].strip().strip('"').split("/")[-1]
    body = [l for l in lines[1:] if not l.startswith('"Function Name"')]
    rd = csv.reader(io.StringIO("\n".join(body)))
    hdr = next(rd)
    i_samp = hdr.index("Warp Stall Sampling (All Samples)")
    stall = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    for r in rd:
        if len(r) <= i_samp or not r[0]:
            continue
        try:
            s = float(r[i_samp] or 0)
        except ValueError:
            continue
        if s <= 0:
            continue
        st = sorted(((float(r[i]), h[6:]) for i, h in stall if r[i] not in ("", "0", "-")), reverse=True)[:3]
        rows.append((s, fname, r[0], r[1].strip()[:60], st))
tot = sum(r[0] for r in rows)
rows.sort(reverse=True)
print(f"total samples {tot:.0f}")
for s, f, ln, src, st in rows[:N]:
    print(f"{100*s/tot:5.1f}% {f}:{ln:>4} {src:60s} " + ", ".join(f"{h}={v:.0f}" for v, h in st))
