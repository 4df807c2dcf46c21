#!/bin/bash
# per-pass detail + ncu full capture of the first 4 passes of a step (after warm-up)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-p2}
timeout 300 python scripts/bench_pass.py --opts "${2:-plan=1}" --detail > gpurun_out/pass_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 63 -c 4 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
