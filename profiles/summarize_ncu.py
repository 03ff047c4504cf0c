"""Summarise an ncu report (or launch-list CSV) into the markdown tables kept under profiles/.

    python profiles/summarize_ncu.py full  gpurun_out/prof.ncu-rep  > profiles/rNN_ncu_full.md
    python profiles/summarize_ncu.py launches gpurun_out/launches.csv > profiles/rNN_launches.md

`full` reads a `ncu --set full` capture (`ncu -i ... --page raw --csv`) and prints, per kernel
launch, duration, DRAM bytes read/written (the roofline `traffic`), achieved DRAM throughput,
SM/issue utilisation and the fp64/fma/tensor pipe activity. `launches` reads the
`--metrics gpu__time_duration.sum --csv` launch list and prints per-kernel totals and shares.
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

FULL_METRICS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "MB rd"),
    ("dram__bytes_write.sum", "MB wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %pk"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %pk"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def _to_mb(v, unit):
    v = float(v)
    u = unit.lower()
    if u.startswith("gbyte"):
        return v * 1e3
    if u.startswith("kbyte"):
        return v * 1e-3
    if u == "byte":
        return v * 1e-6
    return v


def _to_us(v, unit):
    v = float(v)
    u = unit.lower()
    if u in ("ms", "msecond"):
        return v * 1e3
    if u in ("ns", "nsecond"):
        return v * 1e-3
    return v


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(head)}
    print("| # | kernel | " + " | ".join(lbl for _, lbl in FULL_METRICS) + " |")
    print("|---|---|" + "---|" * len(FULL_METRICS))
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        cells = []
        for m, lbl in FULL_METRICS:
            if m not in col or r[col[m]] == "":
                cells.append("n/a")
                continue
            v, u = r[col[m]], units[col[m]]
            try:
                if lbl.startswith("MB"):
                    cells.append(f"{_to_mb(v.replace(',', ''), u):.2f}")
                elif lbl == "us":
                    cells.append(f"{_to_us(v.replace(',', ''), u):.1f}")
                elif "%" in lbl:
                    cells.append(f"{float(v.replace(',', '')):.1f}")
                else:
                    cells.append(v)
            except ValueError:
                cells.append(v)
        print(f"| {r[col['ID']]} | `{name}` | " + " | ".join(cells) + " |")


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        t = _to_us(r["Metric Value"].replace(",", ""), r.get("Metric Unit", "us"))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(v[1] for v in agg.values()) or 1.0
    print("| kernel | launches | total us | avg us | share |")
    print("|---|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {t:.1f} | {t / n:.1f} | {100 * t / tot:.1f}% |")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
