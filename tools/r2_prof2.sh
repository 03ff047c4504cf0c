#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2g}
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_st0|k_st_sketch|k_st_shrink' -c 4 \
    -o gpurun_out/${tag}_c5 python bench.py --config c5 --steps 1 --warmup 0 --e2e-steps 0 --decompose 0 --no-cpu-baseline \
    > gpurun_out/${tag}_c5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_qr_cluster' -c 2 \
    -o gpurun_out/${tag}_c4 python bench.py --config c4 --steps 1 --warmup 0 --e2e-steps 0 --decompose 0 --no-cpu-baseline \
    > gpurun_out/${tag}_c4.log 2>&1
echo done
