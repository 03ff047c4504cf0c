cd $GRAFT_REPO_ROOT
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_slab_f32.py -q > gpurun_out/r2k_rep$i.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_rep$i.log; done
