"""Wall time per synchronous evaluation (LABS n=26 p=10) through several
public-API call shapes, to locate host / allocation overheads."""
import os
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
K = 20


def run(name, fn):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(K):
        fn(i)
    torch.cuda.synchronize()
    print(f"{name}: {1e3 * (time.perf_counter() - t0) / K:.3f} ms/eval", flush=True)


def d(i):
    r = sim.simulate_qaoa(g + 1e-4 * i, b)
    e = sim.get_expectation(r)
    del r
    return e


run("objective", lambda i: sim.objective(g + 1e-4 * i, b))
run("get_expectation(simulate_qaoa(reuse_buffer=True))",
    lambda i: sim.get_expectation(sim.simulate_qaoa(g + 1e-4 * i, b, reuse_buffer=True)))
run("get_expectation(simulate_qaoa())", lambda i: sim.get_expectation(sim.simulate_qaoa(g + 1e-4 * i, b)))
run("r = simulate_qaoa(); get_expectation(r); del r", d)
run("simulate_qaoa() only, no sync", lambda i: sim.simulate_qaoa(g + 1e-4 * i, b, reuse_buffer=True))
run("objective", lambda i: sim.objective(g + 1e-4 * i, b))
