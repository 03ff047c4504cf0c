#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2stgen}
timeout 900 python -m pytest tests/test_gpu_slab_f32.py tests/test_gpu_loopback.py -q > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
timeout 900 python -m pytest tests/test_gpu_configs.py -q -k "c5 or c3" > gpurun_out/${tag}_cfgtest.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_cfgtest.log
for c in c5 c3; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_$c.log 2>&1; done
timeout 300 python bench.py --config c5 --variant fused --steps 5 --warmup 2 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c5f.log 2>&1
echo done
