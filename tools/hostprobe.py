import time, sys
sys.path.insert(0, '.')
import torch
import paper_1901_01652_b200 as trg
from paper_1901_01652_b200.synthetic import CONFIGS, make_tensor
ctx = trg.default_context()
cfg = CONFIGS['c2']
x, _ = make_tensor(ctx, cfg, seed=0)
spec = trg.ProjectionSpec(cfg['K'], 0)
stream = torch.cuda.ExternalStream(ctx.stream())
def step():
    trg.DeviceSketch(ctx, x, spec).close()
for _ in range(5): step()
ctx.synchronize()
for rep in range(3):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    t0 = time.perf_counter()
    for _ in range(20): step()
    t1 = time.perf_counter()
    ev1.record(stream); ev1.synchronize()
    t2 = time.perf_counter()
    print(f"host enqueue {1e3*(t1-t0)/20:.3f} ms/step, gpu {ev0.elapsed_time(ev1)/20:.3f} ms/step, wall {1e3*(t2-t0)/20:.3f}")
