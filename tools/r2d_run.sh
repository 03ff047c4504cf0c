cd $GRAFT_REPO_ROOT
timeout 120 python tools/tc_debug.py > gpurun_out/r2d_dbg.log 2>&1
echo "rc=$?" >> gpurun_out/r2d_dbg.log
timeout 300 python -m pytest tests/test_gpu_tc.py -q -s > gpurun_out/r2d_tc.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2d_tc.log
