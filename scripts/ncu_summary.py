"""Key metrics + stall reasons + opcode mix + hottest source lines of one ncu report."""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
kid = int(sys.argv[2]) if len(sys.argv) > 2 else 0


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u = raw[0], raw[1]
v = raw[2 + kid]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct"]
for k in keys:
    if k in h:
        i = h.index(k)
        print(f"{k:60s} {v[i][:90]} {u[i]}")
st = []
for i, k in enumerate(h):
    if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
        try:
            st.append((float(v[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(x for x, _ in st) or 1
print("stalls:", ", ".join(f"{k} {x / tot * 100:.0f}%" for x, k in sorted(st, reverse=True)[:8]))
