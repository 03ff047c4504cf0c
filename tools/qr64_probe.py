import sys; sys.path.insert(0, '.')
import numpy as np
import paper_1901_01652_b200 as trg
y = np.random.default_rng(0).standard_normal((1024, 64))
for _ in range(3): trg.economy_q(y)
