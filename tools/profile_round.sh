#!/bin/bash
# Round-end evidence on the GPU box: default bench line, reference arm, ncu launch list and one
# ncu --set full capture of every kernel of one C2 projection step (outputs in gpurun_out/).
cd "$(dirname "$0")/.."
tag=${1:-r1}
python bench.py > gpurun_out/bench_${tag}.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${tag}.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/ncu_l_${tag}.log 2>&1
ncu --set full --import-source on --clock-control none -k 'regex:k_sketch_l1|k_ttm_qreg|k_cqr_fused|k_slab2' -c 12 \
    -o gpurun_out/prof_${tag} python bench.py --steps 1 --warmup 0 --e2e-steps 0 --decompose 0 --no-cpu-baseline \
    > gpurun_out/ncu_f_${tag}.log 2>&1
echo done
