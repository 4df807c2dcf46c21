#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2j}
timeout 600 python scripts/bench_pass.py --n 30 --p 10 --steps 2 --opts "cost_l2=-1,0,1" > gpurun_out/pass_n30cl2_$T.log 2>&1
timeout 600 python scripts/bench_pass.py --n 26 --p 10 --steps 10 --opts "cost_l2=0,1,0,1" > gpurun_out/pass_n26cl2_$T.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_pass16 -s 1 -c 3 --csv --log-file gpurun_out/traffic_n30_$T.csv python scripts/bench_pass.py --n 30 --p 10 --steps 1 --opts "plan=-1" > gpurun_out/ncu_n30_$T.log 2>&1
echo done
