#!/bin/bash
# Lane-butterfly programs (K_LANE3) for 9-target high groups: parity + n=29/30 timing.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2h}
timeout 900 python -m pytest tests/test_gpu_plans.py tests/test_gpu_full_size.py tests/test_gpu_qaoa.py -q -x > gpurun_out/pytest_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$T.log
timeout 600 python scripts/bench_pass.py --n 30 --p 10 --steps 2 --opts "lane3=1,0" --detail > gpurun_out/pass_n30_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --n 29 --p 10 --steps 3 --opts "lane3=1,0" --detail > gpurun_out/pass_n29_$T.log 2>&1
timeout 300 python scripts/bench_pass.py --n 26 --p 10 --steps 10 --opts "lane3=1,0" > gpurun_out/pass_n26_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --n 30 --p 10 --steps 2 --state c64 --opts "lane3=1,0" > gpurun_out/pass_n30c64_$T.log 2>&1
echo done
