#!/bin/bash
# A/B: main vs variant $1 (complex64 occupancy), c64 n=26 p=10, n=30 p=4, n=33 p=2; parity with the variant.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
V=$1; T=${2:-ab3}
for rep in 1 2; do
  for var in "" "$V"; do
    echo "== variant '${var:-main}' rep $rep" >> gpurun_out/ab_$T.log
    FQ_LIB_VARIANT=$var timeout 300 python scripts/bench_pass.py --n 26 --p 10 --steps 20 --state c64 --opts "plan=-1" 2>&1 | grep '"phase"' >> gpurun_out/ab_$T.log
  done
done
for var in "" "$V"; do
  echo "== variant '${var:-main}' large n" >> gpurun_out/ab_$T.log
  FQ_LIB_VARIANT=$var timeout 300 python scripts/bench_pass.py --n 30 --p 4 --steps 3 --state c64 --opts "plan=-1" 2>&1 | grep '"phase"' >> gpurun_out/ab_$T.log
  FQ_LIB_VARIANT=$var timeout 600 python scripts/bench_pass.py --n 33 --p 2 --steps 1 --state c64 --opts "plan=-1" 2>&1 | grep '"phase"' >> gpurun_out/ab_$T.log
done
FQ_LIB_VARIANT=$V timeout 1200 python -m pytest tests/test_gpu_c64.py tests/test_gpu_plans.py -q -x > gpurun_out/pytest_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$T.log
echo done
