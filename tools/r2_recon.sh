#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2rc}
timeout 900 python -m pytest tests/test_gpu_recon.py tests/test_gpu_parity.py -q -x > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
for c in c2 c1 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${tag}_$c.log 2>&1
done
TRG_RECON_SIMT=1 timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${tag}_c2_simt.log 2>&1
echo done
