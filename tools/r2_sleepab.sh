#!/bin/bash
# A/B: sleeping producer/generator waits (libtrg.so) against plain polling (libtrg_poll.so), C3/C5/C4
cd $GRAFT_REPO_ROOT
tag=${1:-r2slp}
for rep in 1 2; do
for v in new poll; do
  if [ $v = new ]; then unset TRG_LIB_PATH; else export TRG_LIB_PATH=$GRAFT_REPO_ROOT/paper_1901_01652_b200/libtrg_poll.so; fi
  for c in c3 c5 c4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_${v}_${c}_$rep.log 2>&1
  done
done; done
echo done
