set -x
touch paper_1901_01652_b200/csrc/stream_f64.cu
TRG_EXTRA_NVCC="-DTRG_SK_PROF" python -c "import sys; sys.path.insert(0,'.'); from paper_1901_01652_b200 import build; build.build()" > /dev/null 2>&1
python bench.py --steps 2 --warmup 1 --e2e-steps 0 --decompose 0 --no-cpu-baseline 2>&1 | grep sk_prof | tail -2
touch paper_1901_01652_b200/csrc/stream_f64.cu
TRG_EXTRA_NVCC="-DTRG_SK_PROF -DTRG_SK_NOGEN" python -c "import sys; sys.path.insert(0,'.'); from paper_1901_01652_b200 import build; build.build()" > /dev/null 2>&1
python bench.py --steps 2 --warmup 1 --e2e-steps 0 --decompose 0 --no-cpu-baseline 2>&1 | grep sk_prof | tail -2
touch paper_1901_01652_b200/csrc/stream_f64.cu
TRG_EXTRA_NVCC="-DTRG_SK_PROF -DTRG_SK_NOMMA" python -c "import sys; sys.path.insert(0,'.'); from paper_1901_01652_b200 import build; build.build()" > /dev/null 2>&1
python bench.py --steps 2 --warmup 1 --e2e-steps 0 --decompose 0 --no-cpu-baseline 2>&1 | grep sk_prof | tail -2
