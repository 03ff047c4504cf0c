import sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle_ref as orc
import paper_1901_01652_b200 as trg
np.set_printoptions(precision=5, linewidth=200, suppress=True)
dims, K = (4, 7, 300), (4, 1, 5)
rng = np.random.default_rng(sum(dims) + 3 * sum(K))
x = rng.standard_normal(dims).astype(np.float32)
proj, bases, ys = orc.sketch(x.astype(np.float64), K, 11)
got = trg.sketch(x, trg.ProjectionSpec(list(K), 11))
print("Y2 got[:4]\n", got.sketches[2][:4], "\nwant[:4]\n", ys[2][:4])
# host P^(2) and Omega_2: D_2 = 4*300*1 (mode 1 columns x K_1), rows 4
P2 = orc.mode_n_product(x.astype(np.float64), 1, bases[1].T)
X2 = orc.unfold(P2, 2)
for D in [1200, 1199, 1201, 1196]:
    om = np.stack([orc.gaussian(11, 4, skip=D + 4 * k) for k in range(5)], axis=1)
    print(D, "host Y2[:2]", (X2 @ om)[:2])
print("Y1 err", np.linalg.norm(got.sketches[1] - ys[1]) / np.linalg.norm(ys[1]))
