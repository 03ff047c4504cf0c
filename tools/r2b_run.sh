cd $GRAFT_REPO_ROOT
rm -f gpurun_out/r2b_parity.jsonl
TRG_PARITY_OUT=gpurun_out/r2b_parity.jsonl timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -s > gpurun_out/r2b_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_gputest.log
