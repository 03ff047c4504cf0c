#!/bin/bash
# C2: where the mode-1 test-matrix unit blocks are generated (spare CTAs of the mode-0 QR launch,
# fewer of them, or the side stream)
cd $GRAFT_REPO_ROOT
tag=${1:-r2omab}
for rep in 1 2; do
timeout 300 python bench.py --steps 300 --warmup 10 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_base_$rep.log 2>&1
TRG_QR_GEN_CTAS=64 timeout 300 python bench.py --steps 300 --warmup 10 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_g64_$rep.log 2>&1
TRG_QR_GEN_CTAS=32 timeout 300 python bench.py --steps 300 --warmup 10 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_g32_$rep.log 2>&1
TRG_SIDE_OMEGA=1 timeout 300 python bench.py --steps 300 --warmup 10 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_side_$rep.log 2>&1
done
echo done
