"""profiles/r1_configs.json from per-config bench logs (development aid).

    python tools/configs_summary.py TAG > profiles/r1_configs.json

reads gpurun_out/cfg_cN_TAG.log (N = 1, 3, 4, 5) and gpurun_out/bench_TAG.log (C2, the bench line).
"""
import json
import sys


def line(path):
    for ln in open(path):
        if ln.startswith("{"):
            return json.loads(ln)
    return None


def main(tag):
    out = {"_command": "python bench.py --config cN --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline "
                       "(C2: the default bench line)", "configs": {}}
    for c in ["c1", "c2", "c3", "c4", "c5"]:
        d = line(f"gpurun_out/bench_{tag}.log" if c == "c2" else f"gpurun_out/cfg_{c}_{tag}.log")
        if d is None:
            continue
        dec = d.get("decompose_e2e") or {}
        out["configs"][c] = {
            "workload": d["config"]["workload"],
            "ms_per_step": d["ms_per_step"],
            "GB_s_of_X": d["value"],
            "stage_roofline_frac": d["stage_roofline"]["frac"],
            "dominant_kernel_roofline": {k: d["roofline"][k] for k in ("kernel", "achieved", "frac")},
            "kernels_us": {k: round(v["avg_ms"] * 1e3, 1) for k, v in d["kernels"].items()},
            "decompose_e2e_s": dec.get("seconds"),
            "decompose_stage_ms": dec.get("stage_ms"),
            "clocks": d.get("clocks"),
        }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
