#!/bin/bash
# n=30 heavy lane passes: prefetch variants + ncu of one heavy and one light pass.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2i}
timeout 600 python scripts/bench_pass.py --n 30 --p 10 --steps 2 --opts "prefetch=-1,1,2;zigzag=1,0" > gpurun_out/pass_n30pf_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass16 -s 1 -c 3 -o gpurun_out/prof_n30_$T python scripts/bench_pass.py --n 30 --p 10 --steps 1 --opts "plan=-1" > gpurun_out/ncu_n30_$T.log 2>&1
echo done
