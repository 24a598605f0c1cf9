"""Hottest CUDA source lines (instructions executed, stall samples) of kernel #k in an ncu report."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kid = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-id", f"::regex:.*:{kid + 1}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur = None
res = []
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 8 and r[0].isdigit() and r[2] == "-":
        try:
            res.append((int(r[7] or 0), int(r[4] or 0), cur, r[0], r[1][:100]))
        except ValueError:
            pass
tot = sum(x[0] for x in res) or 1
tots = sum(x[1] for x in res) or 1
for x in sorted(res, reverse=True)[:top]:
    print(f"{x[0] / tot * 100:5.1f}% inst {x[1] / tots * 100:5.1f}% stall  {x[2]}:{x[3]}  {x[4]}")
