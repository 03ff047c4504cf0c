#!/bin/bash
# small-solve phase split (TRG_SOLVE_PROF=1) on C4/C3 + the GPU suite and a default bench line on this build
cd $GRAFT_REPO_ROOT
tag=${1:-r2sp}
mkdir -p gpurun_out
for c in c4 c3; do
  TRG_SOLVE_PROF=1 timeout 300 python tools/decprof.py $c > gpurun_out/${tag}_${c}.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_gputest.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.log 2>&1
echo done
