#!/bin/bash
# A/B: main vs variant $1 on the XY mixers (bench_xy: ring / complete, c128 / c64), then XY parity.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
V=$1; T=${2:-ab4}
for rep in 1 2; do
  for var in "" "$V"; do
    echo "== variant '${var:-main}' rep $rep" >> gpurun_out/ab_$T.log
    FQ_LIB_VARIANT=$var timeout 300 python scripts/bench_xy.py >> gpurun_out/ab_$T.log 2>&1
  done
done
timeout 1200 python -m pytest tests/test_gpu_full_size.py tests/test_gpu_qaoa.py tests/test_gpu_c64.py tests/test_gpu_sharded_fused.py -q -x > gpurun_out/pytest_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$T.log
echo done
