#!/bin/bash
# Runtime sweep of the mode-0 sketch tile width (TRG_SK_CT) on the GPU box.
cd "$(dirname "$0")/.."
for ct in ${@:-32 64 48 16}; do
  TRG_SK_CT=$ct python bench.py --config c2 --steps 30 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('ct=$ct', 'step_ms', round(d['ms_per_step'],4), 'sketch_m0_us', round(d['kernels']['sketch_m0']['avg_ms']*1000,1))"
done
