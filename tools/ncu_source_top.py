"""Top source lines by warp-stall samples from `ncu --page source --csv --print-source sass,cuda`
(or cuda only).  usage: python tools/ncu_source_top.py file.csv [N]"""
import csv, io, sys

path = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
text = open(path).read()
blocks = text.split('"File Path",')
rows = []
for blk in blocks[1:]:
    lines = blk.splitlines()
    fname = lines[0].strip().strip('"')
    body = "\n".join(l for l in lines[1:] if not l.startswith('"Function Name"'))
    rd = csv.reader(io.StringIO(body))
    hdr = next(rd)
    try:
        i_line = hdr.index("Line No")
        i_src = hdr.index("Source")
        i_samp = hdr.index("Warp Stall Sampling (All Samples)")
    except ValueError:
        continue
    stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    for r in rd:
        if len(r) <= i_samp:
            continue
        try:
            s = float(r[i_samp] or 0)
        except ValueError:
            continue
        if s <= 0:
            continue
        st = sorted(((float(r[i] or 0), h[6:]) for i, h in stall_cols if r[i] not in ("", "0")), reverse=True)[:3]
        rows.append((s, fname.split("/")[-1], r[i_line], r[i_src].strip()[:70], st))
tot = sum(r[0] for r in rows)
rows.sort(reverse=True)
print(f"total samples {tot:.0f}")
for s, f, ln, src, st in rows[:N]:
    print(f"{100*s/tot:5.1f}% {f}:{ln:>4} {src:70s} " + ", ".join(f"{h}={v:.0f}" for v, h in st))
