"""Per-kernel share of an `ncu --metrics gpu__time_duration.sum --csv` launch list.
usage: python tools/launch_summary.py launches.csv [title]"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[i]
ik, iv, im, iu = (hdr.index(c) for c in ('Kernel Name', 'Metric Value', 'Metric Name', 'Metric Unit'))
scale = {'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'nsecond': 1e-3}
t = collections.defaultdict(list)
for r in rows[i + 1:]:
    if len(r) > iv and r[im] == 'gpu__time_duration.sum':
        t[r[ik].split('(')[0].replace('void ', '')].append(float(r[iv].replace(',', '')) * scale.get(r[iu], 1.0))
tot = sum(sum(v) for v in t.values())
print("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches) --")
print((sys.argv[2] if len(sys.argv) > 2 else "") + " -- compare SHARES, not absolutes.\n")
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:48]:48s} launches {len(v):4d}  mean {sum(v)/len(v):8.2f} us  share {100*sum(v)/tot:5.1f}%")
