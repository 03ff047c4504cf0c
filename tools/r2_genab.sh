#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2gab}
for rep in 1 2; do
for v in def g8 g12 g24; do
  if [ $v = def ]; then unset TRG_LIB_PATH; else export TRG_LIB_PATH=$GRAFT_REPO_ROOT/paper_1901_01652_b200/libtrg_$v.so; fi
  timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_${v}_$rep.log 2>&1
done; done
echo done
