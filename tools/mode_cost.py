"""Development: in-step cost of the later modes of C2, by skipping them (K_n = I_n consumes no
draws and launches nothing for mode n). Prints ms per projection for each K."""
import sys

sys.path.insert(0, ".")
import torch

import paper_1901_01652_b200 as trg
from paper_1901_01652_b200.synthetic import CONFIGS, make_tensor

cfg = CONFIGS["c2"]
ctx = trg.default_context()
x, _ = make_tensor(ctx, cfg, seed=0)
stream = torch.cuda.ExternalStream(ctx.stream())
for K in ([16, 16, 16, 16], [16, 16, 16, 100], [16, 16, 100, 100], [16, 100, 100, 100]):
    spec = trg.ProjectionSpec(K, 0)
    for _ in range(5):
        trg.DeviceSketch(ctx, x, spec).close()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(100):
        trg.DeviceSketch(ctx, x, spec).close()
    e1.record(stream)
    e1.synchronize()
    print(K, round(e0.elapsed_time(e1) / 100, 4), "ms")
