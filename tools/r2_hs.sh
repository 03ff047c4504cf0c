#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2x}
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_facade.py -q -x > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
for c in c4 c5; do timeout 900 python bench.py --config $c --steps 5 --warmup 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${tag}_cfg_$c.log 2>&1; done
echo done
