#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2n}
timeout 900 python -m pytest tests/test_gpu_slab_f32.py tests/test_gpu_loopback.py tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
for c in c3 c5; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > /dev/null 2>&1
done
for c in c3 c4 c5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${tag}_cfg_$c.log 2>&1; done
echo done
