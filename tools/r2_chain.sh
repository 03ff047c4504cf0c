#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2chain}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "fused" > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
timeout 300 python bench.py --config c5 --variant fused --steps 5 --warmup 2 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c5f.log 2>&1
TRG_NO_CHAIN01=1 timeout 300 python bench.py --config c5 --variant fused --steps 5 --warmup 2 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c5f_off.log 2>&1
echo done
