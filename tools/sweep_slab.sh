#!/bin/bash
# slab kernel variant sweep (rebuilds slab_tma.cu per variant): arguments are nvcc flag strings
cd "$(dirname "$0")/.."
for fl in "$@"; do
  touch paper_1901_01652_b200/csrc/slab_tma.cu
  TRG_EXTRA_NVCC="$fl" python -c "import sys; sys.path.insert(0,'.'); from paper_1901_01652_b200 import build; build.build()" > /dev/null 2>&1 || { echo "$fl build failed"; continue; }
  python bench.py --steps 20 --warmup 5 --e2e-steps 0 --decompose 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$fl', 'step_ms', round(d['ms_per_step'],4), {k:round(v['avg_ms']*1e3,1) for k,v in d['kernels'].items() if k.endswith(('m1','m2','m3'))})"
done
touch paper_1901_01652_b200/csrc/slab_tma.cu
python -c "import sys; sys.path.insert(0,'.'); from paper_1901_01652_b200 import build; build.build()" > /dev/null 2>&1
