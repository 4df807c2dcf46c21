#!/bin/bash
# A/B: main build vs variant $1, alternating, LABS n=26 p=10 (c128, c64) and n=30 p=10.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
V=$1; T=${2:-ab2}
for rep in 1 2; do
  for var in "" "$V"; do
    echo "== variant '${var:-main}' rep $rep" >> gpurun_out/ab_$T.log
    FQ_LIB_VARIANT=$var timeout 300 python scripts/bench_pass.py --n 26 --p 10 --steps 20 --opts "plan=-1" >> gpurun_out/ab_$T.log 2>&1
    FQ_LIB_VARIANT=$var timeout 300 python scripts/bench_pass.py --n 26 --p 10 --steps 20 --state c64 --opts "plan=-1" >> gpurun_out/ab_$T.log 2>&1
  done
done
for var in "" "$V"; do
  echo "== variant '${var:-main}' n=30" >> gpurun_out/ab_$T.log
  FQ_LIB_VARIANT=$var timeout 600 python scripts/bench_pass.py --n 30 --p 10 --steps 2 --opts "plan=-1" >> gpurun_out/ab_$T.log 2>&1
done
