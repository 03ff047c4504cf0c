#!/bin/bash
# A/B of two libtrg builds: launch lists of every config (A = libtrg_a.so via TRG_LIB_PATH, B = libtrg.so)
cd $GRAFT_REPO_ROOT
tag=${1:-r2ab}
for v in a b; do
  if [ $v = a ]; then export TRG_LIB_PATH=$GRAFT_REPO_ROOT/paper_1901_01652_b200/libtrg_a.so; else unset TRG_LIB_PATH; fi
  for c in c2 c3 c4 c5; do
    timeout 300 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_${v}_$c.log 2>&1
  done
done
echo done
