#!/bin/bash
# ncu --set full of k_st_sketch (C5 sequential mode 1 and C5 fused mode 1)
cd $GRAFT_REPO_ROOT
tag=${1:-r2stn}
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --decompose 0 --no-cpu-baseline"
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_st_sketch" -c 1 -o gpurun_out/${tag}_c5 $B --config c5 > gpurun_out/${tag}_c5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_st_sketch" -c 1 -o gpurun_out/${tag}_c5f $B --config c5 --variant fused > gpurun_out/${tag}_c5f.log 2>&1
echo done
