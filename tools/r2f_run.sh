cd $GRAFT_REPO_ROOT
c=c4
python bench.py --config $c --steps 1 --warmup 0 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/r2f_plain_$c.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tc_sketch -c 1 -o gpurun_out/r2i_prof_$c \
  python bench.py --config $c --steps 1 --warmup 0 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/r2i_ncu_$c.log 2>&1
