cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "u1_one or omega or sketch_f64" > gpurun_out/r2j_test.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_test.log
for i in 1 2; do timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline --decompose 0 | grep '^{' > gpurun_out/r2j_c2_c$i.log; done
