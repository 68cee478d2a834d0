"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel time of the last frame."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
hdr = None
data = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
n = len(data) // frames
agg = collections.OrderedDict()
for d in data[(frames - 1) * n:]:
    k = d["Kernel Name"].split("(")[0][:58]
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"| kernel | launches | us | share |\n|---|---:|---:|---:|")
for k, (c, t) in agg.items():
    print(f"| {k} | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
print(f"| total | {sum(a[0] for a in agg.values())} | {tot:.1f} | |")
