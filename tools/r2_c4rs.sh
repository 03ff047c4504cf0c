#!/bin/bash
# C4 mode-0 tcgen05 sketch: row splits with N-concatenation (fewer MMAs per X block)
cd $GRAFT_REPO_ROOT
tag=${1:-r2c4rs}
B="python bench.py --config c4 --steps 5 --warmup 2 --e2e-steps 0 --decompose 0 --no-cpu-baseline"
timeout 300 $B > gpurun_out/${tag}_c4_def.log 2>&1
TRG_TC_SK_RS=2 TRG_TC_SK_NCAT=1 timeout 300 $B > gpurun_out/${tag}_c4_rs2n.log 2>&1
TRG_TC_SK_RS=4 TRG_TC_SK_NCAT=1 timeout 300 $B > gpurun_out/${tag}_c4_rs4n.log 2>&1
TRG_TC_SK_RS=2 timeout 300 $B > gpurun_out/${tag}_c4_rs2.log 2>&1
TRG_TC_SK_RS=2 TRG_TC_SK_NCAT=1 TRG_TC_SK_STAGE=65536 timeout 300 $B > gpurun_out/${tag}_c4_rs2n64.log 2>&1
timeout 300 $B > gpurun_out/${tag}_c4_def2.log 2>&1
echo done
