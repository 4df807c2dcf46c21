#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2e}
timeout 900 python -m pytest tests/test_gpu_resident.py tests/test_gpu_c64.py tests/test_gpu_qaoa.py -q -x > gpurun_out/pytest_$T.log 2>&1; echo "exit $?" >> gpurun_out/pytest_$T.log
timeout 300 python scripts/bench_xy.py > gpurun_out/xy_$T.log 2>&1
timeout 300 python scripts/latency.py > gpurun_out/latency_$T.log 2>&1
timeout 300 python scripts/res12_probe.py > gpurun_out/res12_$T.log 2>&1
timeout 300 python scripts/bench_configs.py --only 1 --skip-cpu > gpurun_out/config1_$T.log 2>&1
FQ_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --qubits 22 --steps 3 --warmup 3 > gpurun_out/bench_mp2_$T.log 2>&1
echo done
