#!/bin/bash
# TS (A from TMEM) fp32 mode-0 sketch: parity, then C3/C4/C5 against the FFMA / SS kernels
cd $GRAFT_REPO_ROOT
tag=${1:-r2ts}
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/${tag}_test.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_test.log
B="python bench.py --steps 5 --warmup 2 --e2e-steps 0 --decompose 0 --no-cpu-baseline"
for c in c3 c5 c4; do
  TRG_TC_FORCE=1 timeout 300 $B --config $c > gpurun_out/${tag}_${c}_ts.log 2>&1
  TRG_TC_SK_SS=1 TRG_TC_FORCE=1 timeout 300 $B --config $c > gpurun_out/${tag}_${c}_ss.log 2>&1
done
for c in c5 c4 c3; do
  TRG_TC_FORCE=1 TRG_TC_PROF=1 timeout 300 $B --config $c 2>&1 | grep -E "tc_sketch prof" | tail -1 > gpurun_out/${tag}_${c}_ts.txt
done
echo done
