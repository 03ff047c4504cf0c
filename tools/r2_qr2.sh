#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2u}
timeout 600 python -m pytest tests/test_gpu_qr.py -q -x > gpurun_out/${tag}_qrtest.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_qrtest.log
TRG_QR_TRACE=1 timeout 300 python tools/qr_probe_c4.py c4 > gpurun_out/${tag}_qrtrace.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "c3 or c4" > gpurun_out/${tag}_cfgtest.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_cfgtest.log
for c in c3 c4; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > /dev/null 2>&1
done
echo done
