#!/bin/bash
# C2 step time: Gaussian vs Khatri-Rao test matrices, sequential and fused variants
cd "$(dirname "$0")/.."
for v in sequential fused; do for om in gaussian khatri_rao; do
  python bench.py --config ${1:-c2} --variant $v --omega $om --steps 50 --warmup 5 --e2e-steps 0 --decompose 0 \
    --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('$v $om', 'step_ms', round(d['ms_per_step'],4), 'GB/s', round(d['value'],1), ' '.join('%s=%.1f'%(n,k[n]['avg_ms']*1000) for n in k))"
done; done
