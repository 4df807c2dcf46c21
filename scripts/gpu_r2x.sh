#!/bin/bash
# k_pass8 (8 amplitudes x 512 threads for the 7-target fused pass): A/B + parity.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2x}
timeout 600 python scripts/bench_pass.py --n 26 --p 10 --steps 20 --opts "pass8=1,0,1,0" --detail > gpurun_out/pass_p8_$T.log 2>&1
FQ_OPTIONS=pass8=1 timeout 1200 python -m pytest tests/test_gpu_plans.py tests/test_gpu_qaoa.py tests/test_gpu_full_size.py tests/test_gpu_kernels.py tests/test_gpu_properties.py -q -x > gpurun_out/pytest_p8_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_p8_$T.log
timeout 900 ncu --set full --clock-control none -k regex:k_pass8 -c 1 -o gpurun_out/prof_p8_$T python scripts/bench_pass.py --n 26 --p 10 --steps 1 --opts "pass8=1" > gpurun_out/ncu_p8_$T.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_p8_$T.ncu-rep > gpurun_out/p8_summary_$T.txt 2>&1
rm -f gpurun_out/prof_p8_$T.ncu-rep
echo done
