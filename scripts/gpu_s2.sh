#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-s2}
timeout 300 ./scripts/microbench/l2_sweep > gpurun_out/l2_sweep_$T.log 2>&1
timeout 300 python scripts/bench_pass.py --opts "plan=-1" --detail > gpurun_out/pass_$T.log 2>&1
timeout 300 python scripts/host_profile.py > gpurun_out/hostprof_$T.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$T.log
echo done
