#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2tcf}
for c in c3 c5; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_$c.log 2>&1
  TRG_TC_FORCE=1 timeout 300 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_${c}_tc.log 2>&1
done
for r in 2 4; do
TRG_TC_FORCE=1 TRG_TC_SK_STAGE=65536 timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c3_tc_st64.log 2>&1
done
echo done
