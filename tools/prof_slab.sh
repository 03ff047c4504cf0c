#!/bin/bash
# Development: CTA-0 phase cycles of the slab kernels (rebuilds slab_tma.cu with -DTRG_SLAB_PROF).
cd "$(dirname "$0")/.."
touch paper_1901_01652_b200/csrc/slab_tma.cu
TRG_EXTRA_NVCC="-DTRG_SLAB_PROF $SLAB_EXTRA" python -c "import sys; sys.path.insert(0,'.'); from paper_1901_01652_b200 import build; build.build()" > /dev/null 2>&1
python bench.py --steps 1 --warmup 1 --e2e-steps 0 --decompose 0 --no-cpu-baseline 2>&1 | grep slab_ | tail -6
touch paper_1901_01652_b200/csrc/slab_tma.cu
python -c "import sys; sys.path.insert(0,'.'); from paper_1901_01652_b200 import build; build.build()" > /dev/null 2>&1
