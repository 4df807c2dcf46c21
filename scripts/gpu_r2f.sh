#!/bin/bash
# TMA-staged tile loads (option stage): timing A/B, then the GPU suite with staging on every pass.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$T.txt 2>&1
timeout 600 python scripts/bench_pass.py --opts "stage=0,1" --detail > gpurun_out/pass_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --opts "stage=0,1" --state c64 > gpurun_out/pass_c64_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --n 30 --p 4 --opts "stage=0,1" > gpurun_out/pass_n30_$T.log 2>&1
FQ_OPTIONS=stage=1 timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_stage1_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_stage1_$T.log
echo done
