"""profiles/ncu_fresh_traffic.json from an `ncu --set full` capture of fresh_kernel, keyed to
the current kernel source hash (bench.py reads it only while the hash matches).
usage: python tools/fresh_traffic_json.py report.ncu-rep summary_path"""
import csv, io, json, os, subprocess, sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (kernel_src_sha only; bench runs nothing at import)

rep, summary = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, r = rows[0], rows[1], rows[2]


def val(name):
    i = hdr.index(name)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[i]]
    return float(r[i].replace(",", "")) * scale


rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
kname = r[hdr.index("Kernel Name")]
out = {
    "kernel": kname.split("(")[0].replace("void ", "").replace("<unnamed>::", ""),
    "config": "long-video layer (bench.py --profile)",
    "dram_bytes_read_per_launch": int(rd),
    "dram_bytes_write_per_launch": int(wr),
    "dram_bytes_per_launch": int(rd + wr),
    "algorithmic_bytes_per_launch": 38556880,
    "source": f"ncu --set full --clock-control none, {summary}",
    "src_sha": bench.kernel_src_sha(),
}
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                 "ncu_fresh_traffic.json"), "w"), indent=1)
print(json.dumps(out))
