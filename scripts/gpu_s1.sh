#!/bin/bash
# session: A/B of the fused-pass variants, then the GPU test suite, bench, host overhead
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-s1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$T.txt 2>&1
timeout 300 python scripts/bench_pass.py --opts "cost_async=1,0" --detail > gpurun_out/pass_$T.log 2>&1
FQ_LIB_VARIANT=nopair timeout 300 python scripts/bench_pass.py --opts "cost_async=1,0" --detail > gpurun_out/pass_nopair_$T.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$T.log 2>&1
timeout 120 python scripts/host_overhead.py > gpurun_out/host_$T.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$T.log
echo done
