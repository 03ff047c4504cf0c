cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_slab_f32.py tests/test_gpu_tc.py tests/test_gpu_loopback.py tests/test_gpu_parity.py -q -x > gpurun_out/r2k_test.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2k_test.log
for c in c3 c4 c5; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline --decompose 0 > gpurun_out/r2e_cfg_$c.log 2>&1; done
