#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2t3}
TRG_TAIL_TRACE=1 timeout 120 python bench.py --config c2 --steps 3 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c2trace.log 2>&1
TRG_TAIL_TRACE=1 timeout 120 python bench.py --config c1 --steps 3 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c1trace.log 2>&1
TRG_TAIL_TRACE=1 timeout 120 python bench.py --config c5 --steps 3 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c5trace.log 2>&1
TRG_QR_TRACE=1 TRG_TAIL_MB=0 timeout 120 python bench.py --config c4 --steps 1 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c4qr.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tail.py -q -x > gpurun_out/${tag}_tailtest.log 2>&1
for c in c2 c1 c5; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_$c.log 2>&1
  TRG_TAIL_MB=0 timeout 300 python bench.py --config $c --steps 50 --warmup 5 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_${c}_notail.log 2>&1
done
echo done
