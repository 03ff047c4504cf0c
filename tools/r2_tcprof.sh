#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2aa}
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_tc_sketch' -c 1 \
    -o gpurun_out/${tag}_tcsk_c4 python bench.py --config c4 --steps 1 --warmup 0 --e2e-steps 0 --decompose 0 --no-cpu-baseline > /dev/null 2>&1
TRG_TC_FORCE=1 timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_tc_sketch' -c 1 \
    -o gpurun_out/${tag}_tcsk_c3 python bench.py --config c3 --steps 1 --warmup 0 --e2e-steps 0 --decompose 0 --no-cpu-baseline > /dev/null 2>&1
TRG_TC_FORCE=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_c3tc.csv \
    python bench.py --config c3 --steps 2 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > /dev/null 2>&1
echo done
