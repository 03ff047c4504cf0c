#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2gen}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "f32 or c3 or c5 or c4" > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
for c in c5 c3 c4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_$c.log 2>&1
done
echo done
