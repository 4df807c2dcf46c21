#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2o}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_resident8 -s 10 -c 1 -o gpurun_out/prof_res_$T python scripts/res12_probe.py > gpurun_out/ncu_res_$T.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_res_$T.ncu-rep > gpurun_out/res_summary_$T.txt 2>&1
python scripts/ncu_source.py gpurun_out/prof_res_$T.ncu-rep > gpurun_out/res_source_$T.txt 2>&1
ncu -i gpurun_out/prof_res_$T.ncu-rep --page source --csv --print-source sass > gpurun_out/res_sass_$T.csv 2>&1
rm -f gpurun_out/prof_res_$T.ncu-rep
