"""Instruction mix of one kernel in an ncu report: python tools/sass_mix.py rep.ncu-rep ID"""
import collections, csv, subprocess, sys
rep, kid = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-id", f":::{kid}"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
si, ie, st = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
mix, stall = collections.Counter(), collections.Counter()
tot = 0
for r in rows[1:]:
    if len(r) <= max(si, ie, st): continue
    op = r[si].split()[0] if r[si].split() else "?"
    if op.startswith("@"):
        op = r[si].split()[1]
    op = op.split(".")[0]
    if not r[ie].isdigit(): continue
    n = int(r[ie])
    mix[op] += n
    stall[op] += int(r[st] or 0)
    tot += n
print("total warp instructions", tot)
for op, n in mix.most_common(25):
    print(f"{op:10s} {n:12d} {100*n/tot:5.1f}%  stall-samples {stall[op]}")
