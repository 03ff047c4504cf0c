#!/bin/bash
cd $GRAFT_REPO_ROOT
CMD="python bench.py --config c5 --steps 1 --warmup 1 --e2e-steps 0 --decompose 0 --no-cpu-baseline"
$CMD > gpurun_out/c5prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_st_sketch -s 4 -c 1 -o gpurun_out/prof_c5st $CMD > gpurun_out/c5prof_ncu.log 2>&1
echo done
