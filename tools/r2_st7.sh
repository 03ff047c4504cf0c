#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2m}
timeout 600 python -m pytest tests/test_gpu_slab_f32.py tests/test_gpu_loopback.py tests/test_gpu_configs.py -q -x -k "not c3 and not c4" > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_c5.csv \
    python bench.py --config c5 --steps 2 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_st0_sketch|k_st_sketch' -c 2 \
    -o gpurun_out/${tag}_c5 python bench.py --config c5 --steps 1 --warmup 0 --e2e-steps 0 --decompose 0 --no-cpu-baseline \
    > gpurun_out/${tag}_c5.log 2>&1
echo done
