import sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle_ref as orc
import paper_1901_01652_b200 as trg
for dims, K in [((8, 100, 11), (8, 33, 4)), ((4, 7, 300), (4, 1, 5))]:
    rng = np.random.default_rng(sum(dims) + 3 * sum(K))
    x = rng.standard_normal(dims).astype(np.float32)
    proj, bases, ys = orc.sketch(x.astype(np.float64), K, 11)
    got = trg.sketch(x, trg.ProjectionSpec(list(K), 11))
    for n in range(3):
        if K[n] != dims[n]:
            print(dims, n, np.linalg.norm(got.sketches[n] - ys[n]) / np.linalg.norm(ys[n]))
