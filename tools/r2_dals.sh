#!/bin/bash
# device-built ALS systems (device_als_direct): phase split, parity on the configs, decompose timings (device / host LS)
cd $GRAFT_REPO_ROOT
tag=${1:-r2dals}
mkdir -p gpurun_out
for c in c4 c3; do
  TRG_SOLVE_PROF=1 timeout 300 python tools/decprof.py $c > gpurun_out/${tag}_${c}.log 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -x > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
B="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
for c in c4 c3; do
  timeout 600 $B --config $c > gpurun_out/${tag}_${c}_dev.log 2>&1
  TRG_HOST_LS=1 timeout 600 $B --config $c > gpurun_out/${tag}_${c}_host.log 2>&1
done
echo done
