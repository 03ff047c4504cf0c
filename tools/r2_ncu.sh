#!/bin/bash
# ncu --set full captures of one projection per config; the .ncu-rep of C2 and C5 come back, every
# capture also as a details-page CSV (gpurun_out/ is capped at 64 MiB)
cd $GRAFT_REPO_ROOT
tag=${1:-r2w}
cap() {  # name config kernel-regex count
    timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$3" -c $4 \
        -o gpurun_out/${tag}_full_$1 python bench.py --config $2 --steps 1 --warmup 0 --e2e-steps 0 --decompose 0 \
        --no-cpu-baseline > gpurun_out/${tag}_full_$1.log 2>&1
    ncu -i gpurun_out/${tag}_full_$1.ncu-rep --page details --csv > gpurun_out/${tag}_full_$1.csv 2>/dev/null
}
cap c2 c2 'k_sketch_l1|k_ttm_qreg|k_cqr_fused|k_slab2' 12
cap c5 c5 'k_sketch_l1_f32|k_st0|k_st_' 6
cap c4 c4 'k_tc_|k_st_|k_qr_cluster|k_sketch_n' 8
cap c3 c3 'k_sketch_l1_f32|k_tc_|k_st_|k_qr_cluster' 6
rm -f gpurun_out/${tag}_full_c3.ncu-rep gpurun_out/${tag}_full_c4.ncu-rep
du -sh gpurun_out
echo done
