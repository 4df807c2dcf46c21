#!/bin/bash
# One full phase table (option table_full) vs hi x lo tables: A/B + parity.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2u}
timeout 600 python scripts/bench_pass.py --n 26 --p 10 --steps 20 --opts "table_full=1,0,1,0" --detail > gpurun_out/pass_n26tf_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --n 26 --p 10 --steps 20 --state c64 --opts "table_full=1,0,1,0" > gpurun_out/pass_n26c64tf_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --n 30 --p 10 --steps 2 --opts "table_full=1,0" > gpurun_out/pass_n30tf_$T.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_plans.py tests/test_gpu_qaoa.py tests/test_gpu_c64.py tests/test_gpu_full_size.py tests/test_gpu_sharded_fused.py tests/test_gpu_kernels.py -q -x > gpurun_out/pytest_tf_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tf_$T.log
echo done
