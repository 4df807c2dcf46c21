#!/bin/bash
# Per-thread L2 prefetch of the next tile (pf_thread) at n = 30 / 26 / c64.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2m}
timeout 600 python scripts/bench_pass.py --n 30 --p 10 --steps 2 --opts "pf_thread=0,-1,1" --detail > gpurun_out/pass_n30pft_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --n 26 --p 10 --steps 10 --opts "pf_thread=0,1,0,1" > gpurun_out/pass_n26pft_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --n 30 --p 4 --steps 2 --state c64 --opts "pf_thread=0,-1" > gpurun_out/pass_n30c64pft_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --n 32 --p 2 --steps 2 --opts "pf_thread=0,-1" > gpurun_out/pass_n32pft_$T.log 2>&1
echo done
