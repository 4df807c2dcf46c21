#!/bin/bash
# Shared cost tile (cost_stage): A/B timing + parity suites.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2k}
timeout 600 python scripts/bench_pass.py --n 26 --p 10 --steps 10 --opts "cost_stage=1,0,1,0" --detail > gpurun_out/pass_n26cs_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --n 26 --p 10 --steps 10 --state c64 --opts "cost_stage=1,0" > gpurun_out/pass_n26c64cs_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --n 30 --p 10 --steps 2 --opts "cost_stage=1,0" > gpurun_out/pass_n30cs_$T.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_plans.py tests/test_gpu_qaoa.py tests/test_gpu_c64.py tests/test_gpu_kernels.py tests/test_gpu_full_size.py tests/test_gpu_properties.py -q -x > gpurun_out/pytest_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$T.log
echo done
