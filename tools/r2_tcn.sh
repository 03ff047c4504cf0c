#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2tcn}
timeout 600 python -m pytest tests/test_gpu_slab_f32.py -q > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
timeout 900 python -m pytest tests/test_gpu_configs.py -q -k "c4" > gpurun_out/${tag}_c4test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_c4test.log
timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c4.log 2>&1
echo done
