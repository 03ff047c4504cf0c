#!/bin/bash
# compare env variants on C2: each arg "ENV=VAL ..." or "-" for none
cd "$(dirname "$0")/.."
for v in "$@"; do
  for rep in 1 2; do
  env $( [ "$v" = "-" ] || echo $v ) python bench.py --config c2 --steps 100 --warmup 5 --e2e-steps 0 --decompose 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('$v', 'step_ms', round(d['ms_per_step'],4), ' '.join('%s=%.1f'%(n,k[n]['avg_ms']*1000) for n in k))"
  done
done
