"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = defaultdict(lambda: [0, 0.0])
seq = []
for r in rows[hdr + 1:]:
    name = r[ki].split("(")[0].replace("void ", "").replace("mgrc_gpu::dev::", "")[:70]
    us = float(r[vi].replace(",", "")) * scale[r[ui]]
    agg[name][0] += 1
    agg[name][1] += us
    seq.append((name, us))
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if last:
    for n, us in seq[-last:]:
        print(f"{us:10.1f} us  {n}")
    print("----")
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{t:12.1f} us {t / tot * 100:5.1f}%  x{n:<4d} {k}")
