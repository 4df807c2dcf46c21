#!/bin/bash
# Large-n per-pass detail + ncu of the n=30 passes; XY phase share.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2g}
timeout 600 python scripts/bench_pass.py --n 30 --p 10 --steps 2 --opts "plan=-1" --detail > gpurun_out/pass_n30_$T.log 2>&1
timeout 300 python scripts/bench_xy.py > gpurun_out/xy_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass16 -s 3 -c 3 -o gpurun_out/prof_n30_$T python scripts/bench_pass.py --n 30 --p 10 --steps 1 --opts "plan=-1" > gpurun_out/ncu_n30_$T.log 2>&1
echo done
