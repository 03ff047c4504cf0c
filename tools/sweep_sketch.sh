#!/bin/bash
# Variant sweep of the fp64 mode-0 sketch on the GPU box: each argument is
# "CT|extra nvcc flags" (CT = TRG_SK_CT at run time, flags rebuild stream_f64.cu).
cd "$(dirname "$0")/.."
for v in "$@"; do
  ct="${v%%|*}"; fl="${v#*|}"
  touch paper_1901_01652_b200/csrc/stream_f64.cu
  TRG_EXTRA_NVCC="$fl" python -c "import sys; sys.path.insert(0,'.'); from paper_1901_01652_b200 import build; build.build()" > /dev/null 2>&1 || { echo "$v build failed"; continue; }
  TRG_SK_CT=$ct python bench.py --config c2 --steps 30 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', 'step_ms', round(d['ms_per_step'],4), 'sketch_m0_us', round(d['kernels']['sketch_m0']['avg_ms']*1000,1))"
done
touch paper_1901_01652_b200/csrc/stream_f64.cu
python -c "import sys; sys.path.insert(0,'.'); from paper_1901_01652_b200 import build; build.build()" > /dev/null 2>&1
