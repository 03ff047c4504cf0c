#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2zt}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_gputest.log
for i in 1 2; do timeout 300 python bench.py --steps 300 --warmup 10 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c2_$i.log 2>&1; done
TRG_QR_TRACE=1 timeout 120 python bench.py --steps 1 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_qrtrace.log 2>&1
echo done
