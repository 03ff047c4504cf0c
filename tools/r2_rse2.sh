#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2p}
for c in c3 c5; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_rsel_$c.csv python tools/rse_probe.py $c > /dev/null 2>&1
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_rse_f32 -c 1 -o gpurun_out/${tag}_rse_c3 python tools/rse_probe.py c3 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k rse > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
echo done
