#!/bin/bash
# C4 mode-0 tcgen05 sketch: stage size / lo-ring depth sweep
cd $GRAFT_REPO_ROOT
tag=${1:-r2skwr}
run() { timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_$1.log 2>&1; }
run base
TRG_TC_SK_WR=1 run wr1
TRG_TC_SK_WR=1 TRG_TC_SK_STAGE=65536 run wr1_st64
TRG_TC_SK_WR=1 TRG_TC_SK_STAGE=65536 TRG_TC_SK_XR=2 run wr1_st64_xr2
TRG_TC_SK_RS=2 run rs2
TRG_TC_SK_RS=2 TRG_TC_SK_STAGE=65536 TRG_TC_SK_WR=1 run rs2_st64_wr1
TRG_TC_FORCE=1 timeout 300 python -m pytest tests/test_gpu_tc.py -q > gpurun_out/${tag}_tctest.log 2>&1
TRG_TC_SK_WR=1 TRG_TC_SK_STAGE=65536 timeout 600 python -m pytest tests/test_gpu_configs.py -q -k c4 > gpurun_out/${tag}_c4test.log 2>&1
echo done
