#!/bin/bash
# Variant sweep: GPU tests, per-kernel-family pass timing, bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-var}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
timeout 300 python scripts/bench_pass.py --opts "kernel=0,1,2,3" > gpurun_out/pass_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/pass_$TAG.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$TAG.log
echo done
