#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2wide}
timeout 900 python -m pytest tests/test_gpu_slab_f32.py tests/test_gpu_parity.py -q -x -k "f32 or 1000" > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
for rep in 1 2; do
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c3_$rep.log 2>&1
TRG_F32_WIDE=0 timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c3_narrow_$rep.log 2>&1
done
echo done
