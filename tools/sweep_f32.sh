#!/bin/bash
# fp32 mode-0 sketch generator-warp sweep (rebuilds stream_f32.cu per variant): "config|nvcc flags"
cd "$(dirname "$0")/.."
for v in "$@"; do
  cfg="${v%%|*}"; fl="${v#*|}"
  touch paper_1901_01652_b200/csrc/stream_f32.cu
  TRG_EXTRA_NVCC="$fl" python -c "import sys; sys.path.insert(0,'.'); from paper_1901_01652_b200 import build; build.build()" > /dev/null 2>&1 || { echo "$v build failed"; continue; }
  python bench.py --config $cfg --steps 5 --warmup 2 --e2e-steps 0 --decompose 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', 'step_ms', round(d['ms_per_step'],3), 'sketch_m0_us', round(d['kernels']['sketch_m0']['avg_ms']*1000,1))"
done
touch paper_1901_01652_b200/csrc/stream_f32.cu
python -c "import sys; sys.path.insert(0,'.'); from paper_1901_01652_b200 import build; build.build()" > /dev/null 2>&1
