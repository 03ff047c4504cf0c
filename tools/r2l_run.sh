cd $GRAFT_REPO_ROOT
lscpu | head -20 > gpurun_out/r2l_lscpu.txt
rm -f gpurun_out/r2l_parity.jsonl
TRG_PARITY_OUT=gpurun_out/r2l_parity.jsonl timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2l_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2l_gputest.log
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/r2l_cfg_$c.log 2>&1; done
timeout 600 python bench.py > gpurun_out/r2l_bench_c2.log 2>&1
