#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r2y}
timeout 600 python -m pytest tests/test_gpu_resident.py tests/test_gpu_qaoa.py -q -x > gpurun_out/pytest_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$T.log
timeout 300 python scripts/latency.py > gpurun_out/latency_$T.log 2>&1
timeout 300 python - >> gpurun_out/latency_$T.log 2>&1 <<'PY'
import time, numpy as np, torch
from paper_2309_04841_b200 import QaoaSimulator, labs_terms
sim = QaoaSimulator(terms=labs_terms(12))
rng = np.random.default_rng(0); g, b = rng.uniform(0, 1, 4), rng.uniform(0, 1, 4)
for use in (True, False, True, False):
    sim.use_graph = use
    for _ in range(50): sim.objective(g, b)
    t0 = time.perf_counter()
    for _ in range(2000): sim.objective(g, b)
    print(f"objective n=12 p=4 use_graph={use}: {(time.perf_counter() - t0) / 2000 * 1e6:.1f} us/call", flush=True)
PY
echo done
