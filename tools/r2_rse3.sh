#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2r}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_rsel_c3.csv python tools/rse_probe.py c3 > /dev/null 2>&1
TRG_RSE_MT128=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_rsel_c3b.csv python tools/rse_probe.py c3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_rsel_c4.csv python tools/rse_probe.py c4 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k rse > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
echo done
