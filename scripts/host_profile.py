"""Where the host time of one objective evaluation goes (public API,
LABS n=26 p=10): cProfile of simulate_qaoa + get_expectation, plus the GPU
idle gap between back-to-back synchronous evaluations (CUDA events)."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_04841_b200 import QaoaSimulator, labs_terms  # noqa: E402

n, p = int(os.environ.get("N", 26)), 10
rng = np.random.default_rng(0)
g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
sim = QaoaSimulator(terms=labs_terms(n))
for _ in range(3):
    sim.get_expectation(sim.simulate_qaoa(g, b))
torch.cuda.synchronize()
K = 30
# host time inside the API calls (wall) vs device time of the same evaluations
t_sim = t_exp = 0.0
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
t0 = time.perf_counter()
for i in range(K):
    a = time.perf_counter()
    ev[i][0].record()
    r = sim.simulate_qaoa(g, b)
    ev[i][1].record()
    c = time.perf_counter()
    sim.get_expectation(r)
    d = time.perf_counter()
    t_sim += c - a
    t_exp += d - c
wall = (time.perf_counter() - t0) / K
dev = sum(s.elapsed_time(e) for s, e in ev) / K
gaps = [ev[i][0].elapsed_time(ev[i + 1][0]) - ev[i][0].elapsed_time(ev[i][1]) for i in range(K - 1)]
print(f"wall {1e3 * wall:.3f} ms/eval; simulate_qaoa host {1e3 * t_sim / K:.3f} ms; get_expectation (incl. wait) "
      f"{1e3 * t_exp / K:.3f} ms; device span {dev:.3f} ms; start-to-start gap beyond span {np.mean(gaps):.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(K):
    sim.get_expectation(sim.simulate_qaoa(g, b))
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
