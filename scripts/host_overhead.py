"""Host-side cost of one objective evaluation through the public API (LABS
n=26 p=10): enqueue time of simulate_qaoa (no sync), of the raw fused
program (run_program), and the end-to-end time with the scalar read back."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_04841_b200 import QaoaSimulator, labs_terms  # noqa: E402
from paper_2309_04841_b200.mixers import run_program  # noqa: E402

n, p = int(os.environ.get("N", 26)), 10
rng = np.random.default_rng(0)
g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
sim = QaoaSimulator(terms=labs_terms(n))
for _ in range(3):
    sim.get_expectation(sim.simulate_qaoa(g, b))
torch.cuda.synchronize()
K = 20
t0 = time.perf_counter()
res = [sim.simulate_qaoa(g, b, reuse_buffer=True) for _ in range(K)]
t_enq = (time.perf_counter() - t0) / K
torch.cuda.synchronize()
state = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
e = torch.empty(1, dtype=torch.float64, device="cuda")
layers = [(float(x), float(y), 1, 0, n) for x, y in zip(g, b)]
t0 = time.perf_counter()
for _ in range(K):
    run_program(state, n, "x", layers, dc=sim.device_costs, init=True, init_amp=2 ** (-n / 2), expectation_out=e)
t_prog = (time.perf_counter() - t0) / K
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(K):
    sim.get_expectation(sim.simulate_qaoa(g, b))
t_e2e = (time.perf_counter() - t0) / K
print(f"enqueue simulate_qaoa {1e3 * t_enq:.3f} ms, run_program {1e3 * t_prog:.3f} ms, e2e {1e3 * t_e2e:.3f} ms/eval")
