#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2sn64}
timeout 600 python -m pytest tests/test_gpu_slab_f32.py -q > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
TRG_TC_SN_SMALLK=1 timeout 600 python -m pytest tests/test_gpu_slab_f32.py -q > gpurun_out/${tag}_test_smallk.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test_smallk.log
TRG_TC_SN_SMALLK=1 timeout 900 python -m pytest tests/test_gpu_configs.py -q -k c5 > gpurun_out/${tag}_c5test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_c5test.log
for v in 0 1; do
  if [ $v = 1 ]; then export TRG_TC_SN_SMALLK=1; fi
  timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c5_$v.log 2>&1
  timeout 300 python bench.py --config c5 --variant fused --steps 5 --warmup 2 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c5f_$v.log 2>&1
  timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c3_$v.log 2>&1
done
echo done
