#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2ac}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_loopback.py tests/test_gpu_kr.py -q -x > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
for i in 1 2; do timeout 300 python bench.py --steps 300 --warmup 10 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c2_$i.log 2>&1; done
TRG_QR_OMEGA=1 timeout 300 python bench.py --steps 300 --warmup 10 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c2_old.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > /dev/null 2>&1
echo done
