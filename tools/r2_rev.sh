#!/bin/bash
# A/B of the slab kernels' unit order (L2 reuse of P^(1) between ttm_m0 -> sketch_m1 -> ttm_m1), C2
cd $GRAFT_REPO_ROOT
tag=${1:-r2rev}
for rep in 1 2; do
for sk in 0 1; do for tt in 0 1; do
  TRG_REV_SLAB_SK=$sk TRG_REV_SLAB_TTM=$tt timeout 300 python bench.py --steps 300 --warmup 10 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_${sk}${tt}_$rep.log 2>&1
done; done; done
echo done
