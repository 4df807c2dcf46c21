#!/bin/bash
# First-pass cost staging: per-pass A/B (main vs variant built from HEAD), parity.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2w}
for rep in 1 2 3; do
  for var in "" head; do
    echo "== variant '${var:-main}' rep $rep" >> gpurun_out/ab_$T.log
    FQ_LIB_VARIANT=$var timeout 300 python scripts/bench_pass.py --n 26 --p 10 --steps 20 --opts "plan=-1" --detail 2>&1 | grep -E '"phase"|pass  0 |pass 20 ' >> gpurun_out/ab_$T.log
  done
done
timeout 1200 python -m pytest tests/test_gpu_plans.py tests/test_gpu_qaoa.py tests/test_gpu_c64.py tests/test_gpu_full_size.py tests/test_gpu_kernels.py -q -x > gpurun_out/pytest_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$T.log
echo done
