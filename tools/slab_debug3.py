import os, sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle_ref as orc
import paper_1901_01652_b200 as trg
from test_gpu_slab_f32 import CASES
np.set_printoptions(precision=4, linewidth=200, suppress=True)
for dims, K in CASES:
    rng = np.random.default_rng(sum(dims) + 3 * sum(K))
    x = rng.standard_normal(dims).astype(np.float32)
    proj, bases, ys = orc.sketch(x.astype(np.float64), K, 11)
    got = trg.sketch(x, trg.ProjectionSpec(list(K), 11))
    errs = []
    for n in range(len(dims)):
        if K[n] != dims[n]:
            errs.append((n, float(np.linalg.norm(got.sketches[n] - ys[n]) / np.linalg.norm(ys[n]))))
    print(dims, K, errs)
    if max(e for _, e in errs) > 1e-4:
        n = max(errs, key=lambda t: t[1])[0]
        d = got.sketches[n] - ys[n]
        print("bad columns", np.nonzero(np.abs(d).max(axis=0) > 1e-4)[0], "bad rows", np.nonzero(np.abs(d).max(axis=1) > 1e-4)[0][:20], len(np.nonzero(np.abs(d).max(axis=1) > 1e-4)[0]))
