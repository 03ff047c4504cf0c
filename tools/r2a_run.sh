cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
nproc >> gpurun_out/r2a_smi.txt
TRG_FULL_CONFIGS=1 timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/r2a_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a_gputest.log
for c in c3 c4 c5; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2a_cfg_$c.log 2>&1; done
