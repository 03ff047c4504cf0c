#!/bin/bash
# Re-entry check (one GPU): GPU tests, the default bench line, C2 launch list.
cd $GRAFT_REPO_ROOT
tag=${1:-r2chk}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_gputest.log
timeout 600 python bench.py > gpurun_out/${tag}_bench_c2.log 2>&1
timeout 300 python bench.py --steps 300 --warmup 10 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c2_long.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > /dev/null 2>&1
echo done
