#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2t2}
TRG_TAIL_TRACE=1 timeout 120 python bench.py --config c2 --steps 3 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c2trace.log 2>&1
TRG_TAIL_TRACE=1 timeout 120 python bench.py --config c1 --steps 3 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c1trace.log 2>&1
TRG_QR_LEGACY=1 timeout 300 python -m pytest tests/test_gpu_qr.py -q -k "200-32 or 513-33" > gpurun_out/${tag}_qr32.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tail.py -q > gpurun_out/${tag}_tailtest.log 2>&1
echo done
