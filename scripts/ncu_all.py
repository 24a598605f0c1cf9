"""One line per kernel launch of an `ncu --set full` report: duration, DRAM bytes, DRAM % of peak,
occupancy, issue activity and the top stall reasons (the table committed under profiles/)."""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(out)))
h, u = raw[0], raw[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def get(v, k, num=True):
    if k not in h:
        return None
    x = v[h.index(k)]
    if not num:
        return x
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


rows = []
for v in raw[2:]:
    name = get(v, "Kernel Name", False).split("(")[0]
    t = get(v, "gpu__time_duration.sum")
    tu = u[h.index("gpu__time_duration.sum")]
    ms = t / 1e6 if tu == "ns" else (t / 1e3 if tu in ("us", "usecond") else t)
    rb = get(v, "dram__bytes_read.sum") * scale.get(u[h.index("dram__bytes_read.sum")], 1)
    wb = get(v, "dram__bytes_write.sum") * scale.get(u[h.index("dram__bytes_write.sum")], 1)
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                st.append((float(v[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1
    rows.append({"kernel": name, "ms": round(ms, 4), "dram_MB": round((rb + wb) / 1e6, 2),
                 "dram_GBs": round((rb + wb) / (ms * 1e-3) / 1e9, 1) if ms else None,
                 "dram_pct": get(v, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                 "regs": get(v, "launch__registers_per_thread"),
                 "warps_active_pct": get(v, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                 "issue_active_pct": get(v, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                 "stalls": ", ".join(f"{k} {x / tot * 100:.0f}%" for x, k in sorted(st, reverse=True)[:3])})
if len(sys.argv) > 2 and sys.argv[2] == "--json":
    print(json.dumps(rows, indent=1))
else:
    print(f"{'kernel':44s} {'ms':>8s} {'DRAM MB':>9s} {'GB/s':>8s} {'DRAM%':>6s} {'regs':>5s} {'warps%':>7s} {'issue%':>7s}  stalls")
    for r in rows:
        print(f"{r['kernel'][:44]:44s} {r['ms']:8.4f} {r['dram_MB']:9.1f} {r['dram_GBs'] or 0:8.1f} {r['dram_pct'] or 0:6.1f} "
              f"{int(r['regs'] or 0):5d} {r['warps_active_pct'] or 0:7.1f} {r['issue_active_pct'] or 0:7.1f}  {r['stalls']}")
