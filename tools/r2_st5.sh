#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2k}
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_gputest.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_gputest.log
for c in c3 c4 c5; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_st_sketch|k_st_shrink' -c 2 \
    -o gpurun_out/${tag}_c5 python bench.py --config c5 --steps 1 --warmup 0 --e2e-steps 0 --decompose 0 --no-cpu-baseline \
    > gpurun_out/${tag}_c5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_st_sketch|k_st_shrink' -c 2 \
    -o gpurun_out/${tag}_c3 python bench.py --config c3 --steps 1 --warmup 0 --e2e-steps 0 --decompose 0 --no-cpu-baseline \
    > gpurun_out/${tag}_c3.log 2>&1
echo done
