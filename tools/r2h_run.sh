cd $GRAFT_REPO_ROOT
run() { tag=$1; c=$2; shift 2; env "$@" timeout 300 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --decompose 0 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('$tag', '$c', round(d['ms_per_step'],3), 'sk0', round(k['sketch_m0']['avg_ms']*1e3,1), 'ttm0', round(k['ttm_m0']['avg_ms']*1e3,1))" >> gpurun_out/r2h_sweep.log; }
rm -f gpurun_out/r2h_sweep.log
run rs1_3 c4 TRG_TC_SK_RS=1 TRG_TC_SK_NCAT=0
run rs1_3_st16 c4 TRG_TC_SK_RS=1 TRG_TC_SK_NCAT=0 TRG_TC_SK_STAGE=16384
run rs2_3_st16 c4 TRG_TC_SK_RS=2 TRG_TC_SK_NCAT=0 TRG_TC_SK_STAGE=16384
run nottm c5 TRG_NO_TCGEN05=1
