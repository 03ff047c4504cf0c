"""Per-launch DRAM traffic (read + write) of one C2 projection step from an `ncu --set full`
capture (tools/profile_round.sh), written to profiles/ncu_traffic.json for bench.py's
`roofline.traffic`.

    python tools/ncu_traffic.py gpurun_out/prof_r1f.ncu-rep c2 > profiles/ncu_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep, cfg):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    name = head.index("Kernel Name")
    rd, wr = head.index("dram__bytes_read.sum"), head.index("dram__bytes_write.sum")
    out, seen = {}, {"k_slab2_sketch": 0, "k_slab2_ttm": 0}
    for r in rows[2:]:
        kn = r[name]
        if "k_sketch_l1_f64" in kn:
            label = "sketch_m0"
        elif "k_ttm_qreg_f64" in kn:
            label = "ttm_m0"
        elif "k_slab2_sketch" in kn or "k_slab2_ttm" in kn:
            key = "k_slab2_sketch" if "sketch" in kn else "k_slab2_ttm"
            seen[key] += 1
            label = ("sketch_m" if key == "k_slab2_sketch" else "ttm_m") + str(seen[key])
        else:
            continue
        if label in out:
            continue
        b = float(r[rd]) * UNIT.get(units[rd], 1.0) + float(r[wr]) * UNIT.get(units[wr], 1.0)
        out[label] = round(b)
    print(json.dumps({cfg: out, "_source": f"{rep} (ncu --set full --clock-control none, dram__bytes_read.sum + "
                      "dram__bytes_write.sum per launch; ncu flushes L2 before each kernel, so inputs that a "
                      "pipelined step finds in L2 count as DRAM here)"}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "c2")
