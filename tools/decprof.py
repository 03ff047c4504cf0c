import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1901_01652_b200 as trg
from paper_1901_01652_b200.synthetic import CONFIGS, make_tensor
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else 'c2']
ctx = trg.default_context()
x, _ = make_tensor(ctx, cfg, seed=0)
N = len(cfg['dims'])
scfg = trg.SolverConfig(ranks=[cfg['rank']] * N if cfg['method'] == 'als' else None, tolerance=cfg['tol'], max_sweeps=cfg['sweeps'], seed=0)
fn = trg.rtrals if cfg['method'] == 'als' else trg.rtrsvd
fn(x, scfg, trg.ProjectionSpec(cfg['K'], 0))
ctx.synchronize()
ctx.reset_stats(); ctx.set_profiling(True)
t0 = time.perf_counter()
rep = fn(x, scfg, trg.ProjectionSpec(cfg['K'], 0))
ctx.synchronize()
t1 = time.perf_counter()
for lab in ctx.kernel_labels():
    tot, n = ctx.kernel_stats(lab)
    print(f"{lab:16s} {tot:9.3f} ms  x{n}")
print("wall", (t1 - t0) * 1e3, "ms", rep.timings_ms)
