"""Key metrics per kernel of an ncu report: python tools/ncu_sum.py rep.ncu-rep"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
want = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Issue Slots Busy", "Achieved Occupancy",
        "Registers Per Thread", "No Eligible", "L1/TEX Hit Rate", "L2 Hit Rate", "Block Size", "Grid Size",
        "Dynamic Shared Memory Per Block", "Shared Memory Configuration Size"]
cur = None
res = {}
for r in rows[1:]:
    if r[mi] in want:
        res.setdefault((r[ii], r[ki][:60]), {})[r[mi]] = r[vi]
for (i, k), m in res.items():
    print(i, k)
    print("   ", "; ".join(f"{w}={m[w]}" for w in want if w in m))
