#!/bin/bash
cd $GRAFT_REPO_ROOT
CMD="python bench.py --config c2 --steps 1 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline"
$CMD > gpurun_out/tailprof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tail -s 2 -c 1 -o gpurun_out/prof_tail $CMD > gpurun_out/tailprof_ncu.log 2>&1
echo done
