#!/bin/bash
# round 2, session a: validate the (unmeasured) slab sweeps, A/B them, bench, full GPU suite
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > gpurun_out/gpu_$T.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_sweep.py -q -x > gpurun_out/pytest_sweep_$T.log 2>&1; echo "exit $?" >> gpurun_out/pytest_sweep_$T.log
timeout 300 python scripts/bench_pass.py --opts "sweep=1,0" --detail > gpurun_out/pass_$T.log 2>&1
timeout 300 python scripts/bench_pass.py --opts "sweep_team=16,32,37,64" > gpurun_out/pass_team_$T.log 2>&1
timeout 300 python scripts/bench_pass.py --state c64 --opts "sweep=1,0" > gpurun_out/pass_c64_$T.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$T.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$T.log
echo done
