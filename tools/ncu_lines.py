"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo).
usage: python tools/ncu_lines.py report.ncu-rep [kernel-regex] [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
kr = sys.argv[2] if len(sys.argv) > 2 else "."
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kr}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, res, hdr = None, [], None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and r[0] != "Function Name":
        try:
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except Exception:
            continue
        res.append((s, f"{cur_file}:{r[0]}", r[1][:90]))
tot = sum(x[0] for x in res)
print("total samples", tot)
for s, loc, src in sorted(res, reverse=True)[:N]:
    print(f"{s:6d} {100.0*s/max(tot,1):5.1f}% {loc:22s} {src}")
