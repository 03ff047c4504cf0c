#!/bin/bash
# Round-2 final evidence pass on the device-small-solve build (one GPU): GPU tests with parity records, the default
# reference arm, every BASELINE config with e2e + decompose, the fused variant, launch lists, ncu
# --set full captures of C2 and C4 (every ncu run of a call counts as one).
cd $GRAFT_REPO_ROOT
tag=${1:-r2f3}
nvidia-smi > gpurun_out/${tag}_smi.txt 2>&1
rm -f gpurun_out/${tag}_parity.jsonl
TRG_PARITY_OUT=gpurun_out/${tag}_parity.jsonl timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_gputest.log
timeout 900 python bench.py > gpurun_out/${tag}_bench_c2.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_ref.log 2>&1
for c in c1 c3 c4 c5; do timeout 900 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/${tag}_cfg_$c.log 2>&1; done
timeout 600 python bench.py --config c5 --variant fused --steps 10 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > gpurun_out/${tag}_cfg_c5fused.log 2>&1
for c in c2 c4; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --e2e-steps 0 --decompose 0 --no-cpu-baseline > /dev/null 2>&1
done
timeout 900 python bench.py --impl reference --config c4 --steps 1 --warmup 1 > gpurun_out/${tag}_bench_ref_c4.log 2>&1
du -sh gpurun_out
echo done
