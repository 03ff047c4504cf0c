#!/bin/bash
# Persistent-tail check (one GPU): tail tests, the whole GPU suite, per-config bench with and without the tail.
cd $GRAFT_REPO_ROOT
tag=${1:-r2t}
timeout 600 python -m pytest tests/test_gpu_tail.py -x -q > gpurun_out/${tag}_tailtest.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_tailtest.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_gputest.log
for c in c2 c1 c5 c4 c3; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_$c.log 2>&1
  TRG_TAIL_MB=0 timeout 300 python bench.py --config $c --steps 50 --warmup 5 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_${c}_notail.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > /dev/null 2>&1
echo done
