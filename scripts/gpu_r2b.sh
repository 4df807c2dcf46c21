#!/bin/bash
# round 2, session b: host latency, bench (incl. config3/config5 keys), launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2b}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > gpurun_out/gpu_$T.txt 2>&1
timeout 300 python scripts/latency.py > gpurun_out/latency_$T.log 2>&1
timeout 300 python scripts/host_profile.py > gpurun_out/hostprof_$T.log 2>&1
N=12 timeout 300 python scripts/host_profile.py > gpurun_out/hostprof12_$T.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$T.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$T.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-configs > gpurun_out/ncu_launch_$T.log 2>&1
echo done
