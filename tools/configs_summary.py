"""profiles/rN_configs.json from the per-config bench logs of an evidence pass (tools/r2_final.sh).

    python tools/configs_summary.py TAG > profiles/r2_configs.json

reads gpurun_out/TAG_cfg_cN.log (N = 1, 3, 4, 5, and c5fused) and gpurun_out/TAG_bench_c2.log (C2, the
default bench line).
"""
import json
import sys


def line(path):
    try:
        for ln in open(path):
            if ln.startswith("{"):
                return json.loads(ln)
    except FileNotFoundError:
        return None
    return None


def main(tag):
    out = {"_command": "python bench.py --config cN --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline "
                       "(C2: the default bench line; c5fused: --variant fused --e2e-steps 0 --decompose 0)",
           "configs": {}}
    for c in ["c1", "c2", "c3", "c4", "c5", "c5fused"]:
        d = line(f"gpurun_out/{tag}_bench_c2.log" if c == "c2" else f"gpurun_out/{tag}_cfg_{c}.log")
        if d is None:
            continue
        dec = d.get("decompose_e2e") or {}
        out["configs"][c] = {
            "workload": d["config"]["workload"],
            "variant": d["config"].get("variant"),
            "ms_per_step": d["ms_per_step"],
            "GB_s_of_X": d["value"],
            "stage_roofline_frac": d["stage_roofline"]["frac"],
            "stage_alg_bytes": d["stage_roofline"]["alg_bytes"],
            "dominant_kernel_roofline": {k: d["roofline"].get(k) for k in ("kernel", "achieved", "frac")},
            "kernels_us": {k: round(v["avg_ms"] * 1e3, 1) for k, v in d["kernels"].items()},
            "e2e_GB_s": (d.get("e2e") or {}).get("value"),
            "decompose_e2e_s": dec.get("seconds"),
            "decompose_stage_ms": dec.get("stage_ms"),
            "clocks": d.get("clocks"),
        }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
