#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2c}
timeout 900 python -m pytest tests/test_gpu_resident.py tests/test_gpu_qaoa.py tests/test_gpu_properties.py -q -x > gpurun_out/pytest_res_$T.log 2>&1; echo "exit $?" >> gpurun_out/pytest_res_$T.log
timeout 300 python scripts/latency.py > gpurun_out/latency_$T.log 2>&1
timeout 300 python scripts/e2e_gap.py > gpurun_out/e2e_gap_$T.log 2>&1
timeout 300 python scripts/bench_configs.py --only 1 > gpurun_out/config1_$T.log 2>&1
echo done
