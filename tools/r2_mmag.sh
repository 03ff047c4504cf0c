#!/bin/bash
# grouped 3xTF32 MMA issue (one asm block per tile): tcgen05 parity + C3/C4 benches
cd $GRAFT_REPO_ROOT
tag=${1:-r2mg}
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_slab_f32.py tests/test_gpu_parity.py -q -x > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
B="python bench.py --steps 5 --warmup 2 --e2e-steps 0 --decompose 0 --no-cpu-baseline"
timeout 300 $B --config c4 > gpurun_out/${tag}_c4.log 2>&1
timeout 300 $B --config c3 > gpurun_out/${tag}_c3.log 2>&1
TRG_TC_FORCE=1 timeout 300 $B --config c3 > gpurun_out/${tag}_c3tc.log 2>&1
TRG_TC_FORCE=1 timeout 300 $B --config c5 > gpurun_out/${tag}_c5tc.log 2>&1
echo done
