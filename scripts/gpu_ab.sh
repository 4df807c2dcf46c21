#!/bin/bash
# A/B sweep of pass options (no tests): usage gpu_ab.sh TAG "opt=a,b;opt2=c,d"
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-ab}
timeout 600 python scripts/bench_pass.py --opts "$2" > gpurun_out/pass_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/pass_$TAG.log
if [ -n "$3" ]; then timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log; fi
