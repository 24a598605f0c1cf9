"""Writes profiles/ncu_traffic.json: per-kernel DRAM traffic per launch
(dram__bytes_read.sum + dram__bytes_write.sum) from `ncu --set full` reports
of one bench workload:  python scripts/ncu_traffic.py WORKLOAD report.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

out = Path(__file__).resolve().parents[1] / "profiles" / "ncu_traffic.json"
res = json.loads(out.read_text()) if out.exists() else {"workloads": {}}
wl = res.setdefault("workloads", {}).setdefault(sys.argv[1], {"kernels": {}})
for rep in sys.argv[2:]:
    raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                     capture_output=True, text=True).stdout)))
    h, u = raw[0], raw[1]
    for v in raw[2:]:
        name = v[h.index("Kernel Name")].split("(")[0]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rb = float(v[h.index("dram__bytes_read.sum")].replace(",", "")) * scale[u[h.index("dram__bytes_read.sum")]]
        wb = float(v[h.index("dram__bytes_write.sum")].replace(",", "")) * scale[u[h.index("dram__bytes_write.sum")]]
        ms = float(v[h.index("gpu__time_duration.sum")].replace(",", ""))
        wl["kernels"][name] = {"dram_bytes": rb + wb, "dram_read": rb, "dram_write": wb,
                                "ncu_duration": f"{ms} {u[h.index('gpu__time_duration.sum')]}", "report": Path(rep).name}
out.write_text(json.dumps(res, indent=1) + "\n")
print(json.dumps(res, indent=1))
