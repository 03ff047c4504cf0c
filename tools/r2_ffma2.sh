#!/bin/bash
# FFMA2 consumers in the fp32 mode-0 sketch: parity + C3/C5 (C4's K_0 = 64 takes the tcgen05 kernel)
cd $GRAFT_REPO_ROOT
tag=${1:-r2f2}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
B="python bench.py --steps 5 --warmup 2 --e2e-steps 0 --decompose 0 --no-cpu-baseline"
for c in c3 c5; do
  timeout 300 $B --config $c > gpurun_out/${tag}_${c}.log 2>&1
done
timeout 300 $B --config c5 --variant fused > gpurun_out/${tag}_c5fused.log 2>&1
echo done
