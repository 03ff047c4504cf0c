"""Time trg.rse on a BASELINE config's synthetic tensor (development probe).
python tools/rse_probe.py c3"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1901_01652_b200 as trg
from paper_1901_01652_b200 import synthetic as syn

cfg = syn.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
ctx = trg.Context(0)
x, cores = syn.make_tensor(ctx, cfg, 0)
cores = [np.asarray(c) for c in cores]
for rep in range(3):
    t = time.perf_counter()
    r = trg.rse(x, cores, ctx=ctx)
    print(f"rse {r:.9f} wall {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)
