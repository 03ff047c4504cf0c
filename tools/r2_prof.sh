#!/bin/bash
# ncu --set full captures of the fp32 configs' kernels (one projection each)
cd $GRAFT_REPO_ROOT
tag=${1:-r2b}
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_sketch_l1_f32|k_ttm_l1_f32|k_sketch_n_f32|k_ttm_n_f32' -c 6 \
    -o gpurun_out/${tag}_c5 python bench.py --config c5 --steps 1 --warmup 0 --e2e-steps 0 --decompose 0 --no-cpu-baseline \
    > gpurun_out/${tag}_c5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_sketch_l1_f32|k_cqr_small|k_sketch_n_f32|k_ttm_n_f32' -c 5 \
    -o gpurun_out/${tag}_c3 python bench.py --config c3 --steps 1 --warmup 0 --e2e-steps 0 --decompose 0 --no-cpu-baseline \
    > gpurun_out/${tag}_c3.log 2>&1
echo done
