"""Development: wall and stage times of repeated trg_decompose_host calls on a BASELINE config."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1901_01652_b200 as trg
from paper_1901_01652_b200.synthetic import CONFIGS, make_tensor
cfg = CONFIGS[sys.argv[1]]
ctx = trg.default_context()
x, _ = make_tensor(ctx, cfg, seed=0)
N = len(cfg['dims'])
host = torch.empty(int(np.prod(cfg['dims'])), dtype=torch.float64 if cfg['dtype']=='f64' else torch.float32).pin_memory()
host.copy_(torch.from_numpy(np.ascontiguousarray(x.numpy().reshape(-1, order='F'))))
scfg = trg.SolverConfig(ranks=[cfg['rank']] * N if cfg['method'] == 'als' else None, tolerance=cfg['tol'], max_sweeps=cfg['sweeps'], seed=0)
arr = host.numpy().reshape(cfg['dims'], order='F')
for i in range(4):
    t0 = time.perf_counter()
    rep = trg.decompose(arr, cfg['method'], scfg, trg.ProjectionSpec(cfg['K'], 0))
    t1 = time.perf_counter()
    print(i, round((t1-t0)*1e3,2), {k: round(v,2) for k,v in rep.timings_ms.items()})
