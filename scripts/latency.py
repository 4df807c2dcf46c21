"""Single-call latency of one objective evaluation (BASELINE config 1, LABS
n=12 p=4, and the headline n=26 p=10): device time of the fused program
(CUDA events), host enqueue time, and the synchronous wall time of each
public call (simulate_qaoa + get_expectation, objective)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_04841_b200 import QaoaSimulator, labs_terms  # noqa: E402
from paper_2309_04841_b200.mixers import run_program  # noqa: E402


def wall(fn, k):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / k


for n, p, K in ((12, 4, 500), (16, 4, 300), (26, 10, 20)):
    rng = np.random.default_rng(0)
    g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
    sim = QaoaSimulator(terms=labs_terms(n))
    state = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
    e = torch.empty(1, dtype=torch.float64, device="cuda")
    layers = [(float(x), float(y), 1, 0, n) for x, y in zip(g, b)]
    prog = lambda: run_program(state, n, "x", layers, dc=sim.device_costs, init=True,  # noqa: E731
                               init_amp=2 ** (-n / 2), expectation_out=e)
    for _ in range(5):
        prog()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        prog()
    e1.record()
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / K
    t0 = time.perf_counter()
    for _ in range(K):
        prog()
    enq = 1e3 * (time.perf_counter() - t0) / K
    torch.cuda.synchronize()
    api = wall(lambda: sim.get_expectation(sim.simulate_qaoa(g, b)), K)
    obj = wall(lambda: sim.objective(g, b), K)
    prog_sync = wall(lambda: (prog(), e.item()), K)
    print(f"n={n} p={p}: device {dev:.4f} ms/eval back to back; run_program enqueue {enq:.4f} ms; "
          f"run_program+item {prog_sync:.4f} ms; simulate_qaoa+get_expectation {api:.4f} ms; objective {obj:.4f} ms",
          flush=True)
