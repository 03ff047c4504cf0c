#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2skwr2}
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_configs.py tests/test_gpu_parity.py -q -k "tc or c4 or f32" > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
TRG_TC_FORCE=1 timeout 300 python -m pytest tests/test_gpu_tc.py -q > gpurun_out/${tag}_tcforce.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_tcforce.log
for rep in 1 2; do timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c4_$rep.log 2>&1; done
echo done
