#!/bin/bash
# Tile pairs with one 256-B-run prefetch per pair (option pair) at n = 29 / 30 / 32, parity suites.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2t}
timeout 600 python scripts/bench_pass.py --n 30 --p 10 --steps 2 --opts "pair=-1,0,-1,0" > gpurun_out/pass_n30pair_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --n 29 --p 10 --steps 3 --opts "pair=-1,0" > gpurun_out/pass_n29pair_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --n 30 --p 4 --steps 2 --state c64 --opts "pair=-1,0" > gpurun_out/pass_n30c64pair_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --n 32 --p 2 --steps 2 --opts "pair=-1,0" > gpurun_out/pass_n32pair_$T.log 2>&1
FQ_OPTIONS=pair=1 timeout 1200 python -m pytest tests/test_gpu_plans.py tests/test_gpu_qaoa.py tests/test_gpu_c64.py tests/test_gpu_full_size.py tests/test_gpu_sharded_fused.py -q -x > gpurun_out/pytest_pair_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_pair_$T.log
echo done
