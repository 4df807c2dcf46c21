#!/bin/bash
# One GPU session: tests, smoke, bench, per-pass detail, ncu launch list + full capture.  Outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-round}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$TAG.log
timeout 300 python scripts/bench_pass.py --opts "plan=-1" --detail > gpurun_out/pass_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_pass -s 63 -c 21 --csv --log-file gpurun_out/traffic_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_traffic_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 63 -c 4 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full_$TAG.log 2>&1
# extra kernels: complex64 passes, the spanning (sharded, G) pass in-process, the XY pass; all BASELINE configs
timeout 600 python bench.py --state c64 --steps 20 --warmup 5 > gpurun_out/bench_c64_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_pass16<.*float' -s 20 -c 3 -o gpurun_out/prof_c64_$TAG python bench.py --state c64 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_c64_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_pass16<.*bool.1>' -c 2 -o gpurun_out/prof_g_$TAG python scripts/bench_sharded_inprocess.py --n 26 --steps 1 > gpurun_out/ncu_g_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xy_pass -s 17 -c 2 -o gpurun_out/prof_xy_$TAG python scripts/bench_configs.py --only 4 --skip-cpu > gpurun_out/ncu_xy_$TAG.log 2>&1
timeout 1500 python scripts/bench_configs.py > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err
timeout 300 python scripts/bench_xy.py > gpurun_out/xy_$TAG.log 2>&1
timeout 300 python scripts/latency.py > gpurun_out/latency_$TAG.log 2>&1
# the N > 1 path of bench.py end to end as two ranks sharing this one GPU (validation only:
# gloo host collectives, CUDA IPC peer mappings on one device; timings are not meaningful)
FQ_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --qubits 22 --steps 3 --warmup 3 > gpurun_out/bench_mp2_$TAG.log 2>&1
echo done
