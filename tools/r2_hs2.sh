#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2y}
g++ -O3 -march=native -fopenmp -std=c++17 -I paper_1901_01652_b200/csrc tools/dev/hsb_phases.cpp tools/dev/hs_phases.cpp -o /tmp/hsb2 > gpurun_out/${tag}_build.log 2>&1
for t in 16 8 4; do OMP_NUM_THREADS=$t /tmp/hsb2 64 64 32 20 15 > gpurun_out/${tag}_hs_$t.log 2>&1; done
OMP_PROC_BIND=close OMP_PLACES=cores /tmp/hsb2 64 64 32 20 15 > gpurun_out/${tag}_hs_bind.log 2>&1
nproc > gpurun_out/${tag}_nproc.txt; lscpu | grep -E 'Thread|Core|Socket' >> gpurun_out/${tag}_nproc.txt
echo done
