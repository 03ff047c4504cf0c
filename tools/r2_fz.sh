#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2fz}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_gputest.log
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${tag}_c4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${tag}_launches_c5fused.csv \
    python bench.py --config c5 --variant fused --steps 1 --warmup 1 --e2e-steps 0 --decompose 0 --no-cpu-baseline > /dev/null 2>&1
echo done
