#!/bin/bash
# Source-level ncu of the n=26 fused pass; multi-process tests against the oracle.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2l}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass16 -s 44 -c 1 -o gpurun_out/prof_heavy_$T python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_heavy_$T.log 2>&1
python scripts/ncu_source.py gpurun_out/prof_heavy_$T.ncu-rep > gpurun_out/heavy_source_$T.txt 2>&1
ncu -i gpurun_out/prof_heavy_$T.ncu-rep --page source --csv --print-source sass > gpurun_out/heavy_sass_$T.csv 2>&1
rm -f gpurun_out/prof_heavy_$T.ncu-rep
timeout 900 python -m pytest tests/test_gpu_sharded_processes.py -q -x > gpurun_out/pytest_mp_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_mp_$T.log
echo done
