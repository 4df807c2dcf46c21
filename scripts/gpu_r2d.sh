#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2d}
timeout 300 python scripts/bench_xy.py > gpurun_out/xy_$T.log 2>&1
timeout 300 python scripts/bench_float_costs.py > gpurun_out/float_$T.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$T.log
echo done
