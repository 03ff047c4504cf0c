"""QR path + Y conditioning of every mode of a config (development probe).
python tools/qr_probe_c4.py c4"""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1901_01652_b200 as trg
from paper_1901_01652_b200 import synthetic as syn, api

cfg = syn.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
ctx = trg.Context(0)
x, _ = syn.make_tensor(ctx, cfg, 0)
sk = api.DeviceSketch(ctx, x, trg.ProjectionSpec(cfg["K"], 0))
res = sk.result()
for n, y in enumerate(res.sketches):
    s = np.linalg.svd(y, compute_uv=False)
    q, path = trg.economy_q(y, return_path=True)
    print(f"mode {n}: Y {y.shape} cond {s[0] / s[-1]:.3e} path(sketch) {res.qr_householder[n]} path(direct) {path}", flush=True)
for rep in range(3):
    for n, y in enumerate(res.sketches):
        trg.economy_q(y)
