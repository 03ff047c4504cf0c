cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_parity.py -q -x > gpurun_out/r2c_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c_gputest.log
