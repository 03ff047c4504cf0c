#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2s}
for c in c2 c5; do
timeout 300 python bench.py --config $c --variant fused --steps 10 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_fused_$c.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_fused_$c.csv \
    python bench.py --config $c --variant fused --steps 2 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > /dev/null 2>&1
done
echo done
