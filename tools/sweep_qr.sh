#!/bin/bash
# QR reduce-width sweep (rebuilds qr.cu per variant): arguments are nvcc flag strings
cd "$(dirname "$0")/.."
for fl in "$@"; do
  touch paper_1901_01652_b200/csrc/qr.cu
  TRG_EXTRA_NVCC="$fl" python -c "import sys; sys.path.insert(0,'.'); from paper_1901_01652_b200 import build; build.build()" > /dev/null 2>&1 || { echo "$fl build failed"; continue; }
  for i in 1 2; do python bench.py --steps 20 --warmup 5 --e2e-steps 0 --decompose 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$fl', 'step_ms', round(d['ms_per_step'],4), 'qr_us', round(d['kernels']['qr']['avg_ms']*1000,1))"; done
done
touch paper_1901_01652_b200/csrc/qr.cu
python -c "import sys; sys.path.insert(0,'.'); from paper_1901_01652_b200 import build; build.build()" > /dev/null 2>&1
