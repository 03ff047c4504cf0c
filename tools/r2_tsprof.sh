#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2tsp}
B="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline"
for c in c5 c4 c3; do
  TRG_TC_FORCE=1 TRG_TC_PROF=1 timeout 300 $B --config $c 2>&1 | grep -E "tc_sketch prof|tc_stage" | tail -14 > gpurun_out/${tag}_${c}_ts.txt
  TRG_TC_SK_SS=1 TRG_TC_FORCE=1 TRG_TC_PROF=1 timeout 300 $B --config $c 2>&1 | grep -E "tc_sketch prof|tc_stage" | tail -14 > gpurun_out/${tag}_${c}_ss.txt
done
echo done
