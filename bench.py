"""Benchmark: rTRD tensor random projection (sketch + projection) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Metric (BASELINE.json): "rTRD sketch+projection GB/s of X and % HBM roofline;
end-to-end time". One step = one full tensor random projection (all modes:
Gaussian sketch with Omega regenerated on the fly, fixed-order split-K
reduction, CholQR2, TTM shrink, and under sharding the NCCL partial sums) of
the device-resident synthetic tensor, from the first kernel to P and every
Q_n resident in HBM. `value` = bytes of X / (device time per step), whole job
(X is sharded along its last mode across ranks; total work is fixed, so the
scaling is strong). Inputs are larger than L2 (C2: X = 800 MB vs 126 MB L2), so
no L2 flush is needed between steps.

`e2e` is the same metric through the reference-facing C ABI with a pinned
HOST buffer: trg_tensor_upload (H2D of X) + trg_sketch_run + D2H of P and
every Q_n, wall clock per step. `decompose_e2e` times the whole Algorithm 1
(trg_decompose_host: H2D, projection, host small solve, back-projection,
fused final RSE, D2H of the cores) once.

`--impl reference` times the reference algorithm's CPU restatement
(oracle/, the reference itself is unbuildable here: see DESIGN.md) with all
host threads on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rTRD sketch+projection GB/s of X"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="sequential", choices=["sequential", "fused"])
    ap.add_argument("--omega", default="gaussian", choices=["gaussian", "khatri_rao"],
                    help="test matrices: the reference's Gaussian draws, or the opt-in Khatri-Rao products (f4)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--decompose", type=int, default=1, help="also time the full trg_decompose_host once")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def workload_name(name, cfg):
    dims = "x".join(str(d) for d in cfg["dims"])
    meth = "rTR-ALS" if cfg["method"] == "als" else "rTR-SVD"
    snr = "noise-free" if cfg["snr"] is None else f"{cfg['snr']:g} dB"
    return f"{name}: {dims} {cfg['dtype']} TR-rank {cfg['rank']} {snr}, K={cfg['K']}, {meth} sketch+projection"


def alg_bytes(cfg, variant="sequential"):
    """SURVEY §8d minimal algorithmic bytes: 2 S_X + sum_{n>=1} 2 S_P(n) + S_P (sequential),
    2 S_X + S_P (fused). Also returns the per-stage tensor sizes."""
    es = 8 if cfg["dtype"] == "f64" else 4
    dims, K = list(cfg["dims"]), list(cfg["K"])
    sizes = [int(np.prod(dims))]
    cur = list(dims)
    for n in range(len(dims)):
        if K[n] != dims[n]:
            cur[n] = K[n]
            sizes.append(int(np.prod(cur)))
    sx, sp = sizes[0] * es, sizes[-1] * es
    if variant == "fused":
        return 2 * sx + sp, sizes, es
    return 2 * sx + sum(2 * s * es for s in sizes[1:-1]) + sp, sizes, es


def kernel_bytes(cfg, label):
    """Algorithmic bytes of one launch of a labelled kernel (reads of its input tensor
    + writes of its output tensor). A fused "ttm_mN+sketch_mM" launch moves the
    shrink's bytes only (the next sketch reads its tiles on chip)."""
    if "+" in label:
        return kernel_bytes(cfg, label.split("+")[0])
    es = 8 if cfg["dtype"] == "f64" else 4
    dims, K = list(cfg["dims"]), list(cfg["K"])
    cur = list(dims)
    for n in range(len(dims)):
        if K[n] == dims[n]:
            continue
        before = int(np.prod(cur))
        after = before // cur[n] * K[n]
        if label == f"sketch_m{n}":
            return before * es
        if label == f"ttm_m{n}":
            return (before + after) * es
        cur[n] = K[n]
    return None


def kernel_flops(cfg, label):
    """Contraction flops of one launch: 2 * |input| * K_n (sketch or shrink of mode n)."""
    label = label.split("+")[0]
    dims, K = list(cfg["dims"]), list(cfg["K"])
    cur = list(dims)
    for n in range(len(dims)):
        if K[n] == dims[n]:
            continue
        before = int(np.prod(cur))
        if label in (f"sketch_m{n}", f"ttm_m{n}"):
            return 2.0 * before * K[n]
        cur[n] = K[n]
    return None


def fp32_peak():
    """Measured FFMA ceiling (tools/fp32_peak.cu -> profiles/fp32_peak.json), TFLOP/s."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp32_peak.json")) as f:
            d = json.load(f)
        return max(v for k, v in d.items() if k.endswith("_ffma"))
    except Exception:
        return None


def fp64_peak():
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            d = json.load(f)
        return max(v for k, v in d.items() if k.endswith("dmma"))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.15)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(cfg_name, label):
    """dram bytes per launch from the committed ncu --set full summary, if it matches."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(cfg_name, {}).get(label)
    except Exception:
        return None


# ------------------------------------------------------------------ CPU legs (oracle)
def cpu_sample(cfg, budget_s, steps):
    """Bounded sample of the workload for the CPU restatement: leading modes kept, trailing
    modes shrunk (never below K_n), sized from a calibration run to ~budget_s / steps."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ref as orc

    dims, K = list(cfg["dims"]), list(cfg["K"])
    rng = np.random.default_rng(0)

    def shape_for(elems):
        s = list(dims)
        for n in range(len(s) - 1, 0, -1):
            while int(np.prod(s)) > elems and s[n] > max(K[n], 2):
                s[n] = max(K[n], s[n] // 2)
        return s

    def run(shape):
        x = rng.standard_normal(shape)
        if cfg["dtype"] == "f32":
            x = x.astype(np.float32).astype(np.float64)
        t0 = time.perf_counter()
        orc.sketch(x, [min(k, d) for k, d in zip(K, shape)], 0)
        return time.perf_counter() - t0, x.nbytes // (1 if cfg["dtype"] == "f64" else 2)

    calib = shape_for(2_000_000)
    t, _ = run(calib)
    per_elem = t / float(np.prod(calib))
    target = max(int(budget_s / max(steps, 1) / max(per_elem, 1e-12)), int(np.prod(calib)))
    shape = shape_for(min(target, int(np.prod(dims))))
    return orc, shape, run


def cpu_baseline(cfg, budget_s=20.0, steps=1):
    orc, shape, run = cpu_sample(cfg, budget_s, steps)
    threads = os.cpu_count() or 1
    orc.set_threads(threads)
    ts = []
    nbytes = 0
    for _ in range(steps):
        t, nbytes = run(shape)
        ts.append(t)
    sec = float(np.mean(ts))
    out = {"value": nbytes / sec / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
           "sample": f"oracle sketch() of a {'x'.join(map(str, shape))} {cfg['dtype']} tensor "
                     f"(same K, fp64 compute), {steps} run(s), {sec:.3f} s each, OpenMP {threads} threads"}
    # SURVEY §8d's faithful single-thread figure (the reference's Eigen path is single-threaded)
    _, shape1, run1 = cpu_sample(cfg, budget_s / 4.0, 1)
    orc.set_threads(1)
    t1, nb1 = run1(shape1)
    orc.set_threads(threads)
    out["single_thread"] = {"value": nb1 / t1 / 1e9, "unit": "GB/s", "cores": 1, "kind": "port",
                            "sample": f"oracle sketch() of a {'x'.join(map(str, shape1))} tensor, 1 run, "
                                      f"{t1:.3f} s, 1 thread"}
    return out


def cpu_algorithm1(cfg, threads, max_elems=2.0e8):
    """Algorithm 1 end to end on the host restatement (oracle rtrd: sketch, small solve,
    back-projection, final RSE), the CPU figure beside the GPU arm's decompose_e2e. Full size
    when X has at most max_elems elements, else the bounded sample of cpu_sample."""
    orc, shape, _ = cpu_sample(cfg, 20.0, 1)
    if float(np.prod(cfg["dims"])) <= max_elems:
        shape = list(cfg["dims"])
    N = len(shape)
    # the config's tensor family (random TR factors plus noise at the config's SNR), as the GPU arm's
    x = orc.reconstruct_full(orc.random_factors(shape, [cfg["rank"]] * N, 0, cfg["scale"]))
    if cfg.get("snr") is not None:
        x = orc.add_noise(x, cfg["snr"], 1)
    if cfg["dtype"] == "f32":
        x = x.astype(np.float32).astype(np.float64)
    K = [min(k, d) for k, d in zip(cfg["K"], shape)]
    orc.set_threads(threads)
    t0 = time.perf_counter()
    if cfg["method"] == "als":
        rep = orc.rtrd("als", x, K, ranks=[cfg["rank"]] * N, tol=cfg["tol"], max_sweeps=cfg["sweeps"])
    else:
        rep = orc.rtrd("svd", x, K, tol=cfg["tol"])
    sec = time.perf_counter() - t0
    return {"seconds": sec, "cores": threads, "kind": "port", "dims": shape, "final_rse": rep.rse_history[-1],
            "call": "oracle rtrd (rtrals/rtrsvd restatement, sketch.hpp:154-165), fp64, TR factors + noise"}


def reference_arm(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return  # under torchrun only rank 0 times the CPU reference; the others exit 0 without work
    budget = 120.0
    orc, shape, run = cpu_sample(cfg, budget, args.steps + args.warmup)
    threads = os.cpu_count() or 1
    orc.set_threads(threads)
    for _ in range(args.warmup):
        run(shape)
    ts = []
    nbytes = 0
    for _ in range(args.steps):
        t, nbytes = run(shape)
        ts.append(t)
    sec = float(np.mean(ts))
    val = nbytes / sec / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.config, cfg), "dims": cfg["dims"], "K": cfg["K"],
                       "sample_dims": shape, "parallelism": "host CPU (reference restatement)"},
            "cpu_baseline": {"value": val, "unit": "GB/s", "cores": threads, "kind": "port",
                             "sample": f"oracle sketch() of a {'x'.join(map(str, shape))} sample per step"},
            "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    line["algorithm1"] = cpu_algorithm1(cfg, threads)
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def main():
    args = parse()
    from paper_1901_01652_b200.synthetic import CONFIGS

    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        reference_arm(args, cfg)
        return

    import torch

    rank, world, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N`: one process per GPU, launched here the way the driver does
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}")
        import socket

        with socket.socket() as sock:
            sock.bind(("127.0.0.1", 0))
            port = sock.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")

    import paper_1901_01652_b200 as trg
    from paper_1901_01652_b200 import _lib as L
    from paper_1901_01652_b200.synthetic import make_tensor

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [trg.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = trg.Context(local, rank, world, obj[0])
    else:
        ctx = trg.Context(local)
    variant = L.TRG_FUSED if args.variant == "fused" else L.TRG_SEQUENTIAL
    if args.omega == "khatri_rao":
        variant |= L.TRG_OMEGA_KHATRI_RAO

    x, cores = make_tensor(ctx, cfg, seed=0)
    spec = trg.ProjectionSpec(cfg["K"], 0)
    stream = torch.cuda.ExternalStream(ctx.stream())
    x_bytes = int(np.prod(cfg["dims"])) * (8 if cfg["dtype"] == "f64" else 4)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        ctx.synchronize()

    def step():
        trg.DeviceSketch(ctx, x, spec, variant).close()

    for _ in range(args.warmup):
        step()
    barrier()

    # ---- timed region: K steps, device time on the library stream, max over ranks
    launches0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
        barrier()
    launches = ctx.launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = x_bytes / (ms_step * 1e-3) / 1e9

    # ---- per-kernel device times (separate profiled pass over the same K steps)
    ctx.reset_stats()
    ctx.set_profiling(True)
    for _ in range(args.steps):
        step()
    ctx.synchronize()
    kernels = {}
    for lab in ctx.kernel_labels():
        tot, n = ctx.kernel_stats(lab)
        kernels[lab] = {"avg_ms": tot / max(n, 1), "launches_per_step": n / args.steps,
                        "share": None, "total_ms": tot}
    ctx.set_profiling(False)
    prof_total = sum(k["total_ms"] for k in kernels.values()) or 1.0
    for k in kernels.values():
        k["share"] = k["total_ms"] / prof_total
        del k["total_ms"]
    peak, peak_src = measured_peak()
    # dominant kernel among the streaming passes (those with algorithmic bytes)
    cands = [k for k in kernels if kernel_bytes(cfg, k)] or list(kernels)
    dom = max(cands, key=lambda k: kernels[k]["avg_ms"] * kernels[k]["launches_per_step"])
    kb = kernel_bytes(cfg, dom)
    # local bytes per launch under sharding
    kb_local = kb / world if kb else None
    roof = None
    if kb_local:
        ach = kb_local / (kernels[dom]["avg_ms"] * 1e-3) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": ncu_traffic(args.config, dom), "alg_bytes_per_launch": kb_local,
                "avg_launch_ms": kernels[dom]["avg_ms"], "peak_source": peak_src}
        fl = kernel_flops(cfg, dom)
        fp64 = fp64_peak()
        if fl and cfg["dtype"] == "f64" and fp64:
            # the fp64 streaming kernels share the FP64 datapath (DMMA + Box-Muller DFMA): second ceiling
            tf = fl / world / (kernels[dom]["avg_ms"] * 1e-3) / 1e12
            roof["fp64_pipe"] = {"achieved_tflops": tf, "peak_tflops": fp64, "frac": tf / fp64,
                                 "flops_per_launch": fl / world,
                                 "peak_source": "measured (profiles/fp64_peak.json, DMMA m8n8k4 loop)"}
        fp32 = fp32_peak()
        if fl and cfg["dtype"] == "f32" and fp32 and dom == "sketch_m0" and cfg["K"][0] < 32:
            # below K_0 = 32 the fp32 mode-0 sketch runs on the CUDA cores (k_sketch_l1_f32, K_0 FFMA
            # per element; tc_f32.cu's dispatch rule): its second ceiling is the FFMA pipe
            tf = fl / world / (kernels[dom]["avg_ms"] * 1e-3) / 1e12
            roof["fp32_pipe"] = {"achieved_tflops": tf, "peak_tflops": fp32, "frac": tf / fp32,
                                 "flops_per_launch": fl / world,
                                 "peak_source": "measured (profiles/fp32_peak.json, FFMA loop)"}
    b_alg, sizes, es = alg_bytes(cfg, args.variant)
    stage = {"alg_bytes": b_alg, "frac": b_alg / world / (ms_step * 1e-3) / 1e9 / peak,
             "definition": "SURVEY §8d B_alg / per-rank step time / measured HBM peak"}

    # ---- end to end through the C ABI with a pinned host buffer: H2D of X (trg_tensor_upload),
    # the projection (trg_sketch_run) and D2H of P and every Q_n (trg_sketch_projected / _basis),
    # all inside the timed region, wall clock, max over ranks.
    import ctypes

    local_np = x.numpy()
    dt = np.float64 if cfg["dtype"] == "f64" else np.float32
    host = torch.empty(local_np.size, dtype=torch.float64 if dt == np.float64 else torch.float32, pin_memory=True)
    host.numpy()[:] = local_np.reshape(-1, order="F")
    del local_np
    k_arr, k_ptr = L.i64(cfg["K"])
    N = len(cfg["dims"])
    p_out = np.empty(int(np.prod(cfg["K"])), dtype=np.float64)
    q_out = [np.empty(cfg["dims"][n] * cfg["K"][n], dtype=np.float64) for n in range(N)]
    h2d = int(np.prod(x.local_shape)) * (8 if dt == np.float64 else 4)
    d2h = p_out.nbytes + sum(q.nbytes for q in q_out)

    def e2e_step():
        L.call("trg_tensor_upload", x.handle, ctypes.c_void_p(host.data_ptr()))
        h = ctypes.c_void_p()
        L.call("trg_sketch_run", ctx.handle, x.handle, k_ptr, ctypes.c_uint64(0), ctypes.c_int(variant),
               ctypes.byref(h))
        L.call("trg_sketch_projected", h, p_out.ctypes.data_as(L.c_dp))
        for n in range(N):
            L.call("trg_sketch_basis", h, ctypes.c_int(n), q_out[n].ctypes.data_as(L.c_dp))
        L.call("trg_sketch_destroy", h)

    e2e = None
    if args.e2e_steps > 0:
        e2e_step()  # warm-up
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        sec = (time.perf_counter() - t0) / args.e2e_steps
        if dist is not None:
            t = torch.tensor([sec], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sec = float(t.item())
        e2e = {"value": x_bytes / sec / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": sec * 1e3, "steps": args.e2e_steps,
               "call": "C ABI: trg_tensor_upload (pinned host X) + trg_sketch_run + trg_sketch_projected/_basis"}

    # ---- full Algorithm 1 through the C ABI (trg_decompose_host): H2D, projection, host small
    # solve, back-projection, fused final RSE, D2H of the cores. Reported beside e2e.
    decomp = None
    if args.decompose:
        scfg_ranks = [cfg["rank"]] * N if cfg["method"] == "als" else None
        r_arr, r_ptr = L.i64(scfg_ranks) if scfg_ranks else (None, None)
        d_arr, d_ptr = L.i64(cfg["dims"])

        def decompose_once():
            h = ctypes.c_void_p()
            L.call("trg_decompose_host", ctx.handle, ctypes.c_int(L.TRG_F64 if dt == np.float64 else L.TRG_F32),
                   ctypes.c_int(N), d_ptr, ctypes.c_void_p(host.data_ptr()),
                   ctypes.c_int(L.TRG_ALS if cfg["method"] == "als" else L.TRG_SVD), r_ptr,
                   ctypes.c_double(cfg["tol"]), ctypes.c_int64(cfg["sweeps"]), ctypes.c_uint64(0), k_ptr,
                   ctypes.c_uint64(0), ctypes.c_int(variant), ctypes.byref(h))
            return trg.api._report(h, cfg["dims"])

        decompose_once()  # warm-up: first-use kernel loading and allocator growth stay untimed
        barrier()
        t0 = time.perf_counter()
        rep = decompose_once()
        sec = time.perf_counter() - t0
        decomp = {"seconds": sec, "stage_ms": rep.timings_ms, "final_rse": rep.rse_history[-1], "ranks": rep.ranks,
                  "method": "rTR-ALS" if cfg["method"] == "als" else "rTR-SVD",
                  "warmup": 1, "call": "C ABI: trg_decompose_host (pinned host X)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg, args.cpu_budget_s)
        except Exception as exc:  # the baseline must not kill the GPU line
            cpu = {"value": None, "error": str(exc)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic (reference random_factors + "
                "noise at exact SNR, generated on device)",
                "config": {"workload": workload_name(args.config, cfg), "dims": cfg["dims"], "K": cfg["K"],
                           "variant": args.variant, "omega": args.omega, "parallelism": f"last-mode shards x{world}" if world > 1
                           else "single GPU", "l2": "X larger than L2 (no flush needed)"},
                "roofline": roof, "stage_roofline": stage, "cpu_baseline": cpu, "e2e": e2e, "decompose_e2e": decomp,
                "gpu_launches": launches, "clocks": clk.summary(), "kernels": kernels}
        print(json.dumps(line), flush=True)
    barrier()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
