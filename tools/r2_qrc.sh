#!/bin/bash
cd $GRAFT_REPO_ROOT
tag=${1:-r2qrc}
timeout 600 python -m pytest tests/test_gpu_qr.py -q > gpurun_out/${tag}_qrtest.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_qrtest.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_loopback.py -q -x > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
TRG_QR_TRACE=1 timeout 120 python bench.py --config c4 --steps 1 --warmup 2 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_c4qr.log 2>&1
for c in c4 c3; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_$c.log 2>&1
done
echo done
