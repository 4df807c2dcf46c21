"""X-mixer evaluation with a FLOAT-weight diagonal (no uint16 grid: the phase is
sincos(gamma * c) per amplitude, as the reference), n = 26, p = 10: the
portfolio instance of BASELINE config 4 driven by the X mixer, and a random
float polynomial.  Reports evals/s and the per-pass breakdown."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_04841_b200 import QaoaSimulator, TermPolynomial, _lib  # noqa: E402
from paper_2309_04841_b200.problems import portfolio_terms  # noqa: E402

n, p = 26, 10
rng = np.random.default_rng(0)
g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
polys = {"portfolio26": portfolio_terms(n)}
pairs = []
for _ in range(200):
    k = int(rng.integers(1, 5))
    pairs.append((float(rng.uniform(-2, 2)), tuple(sorted(rng.choice(n, k, replace=False).tolist()))))
polys["random_float26"] = TermPolynomial.from_pairs(n, pairs)
for name, poly in polys.items():
    sim = QaoaSimulator(terms=poly)
    for _ in range(2):
        sim.get_expectation(sim.simulate_qaoa(g, b, reuse_buffer=True))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        sim.simulate_qaoa(g, b, reuse_buffer=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    _lib.call("fq_set_option", b"time_passes", 1)
    sim.simulate_qaoa(g, b, reuse_buffer=True)
    info = (ctypes.c_int * (5 * 64))()
    tms = (ctypes.c_float * 64)()
    cnt = _lib.load().fq_last_passes(info, tms, 64)
    _lib.call("fq_set_option", b"time_passes", 0)
    kinds = {}
    for i in range(cnt):
        key = (info[5 * i], info[5 * i + 1])
        kinds.setdefault(key, []).append(tms[i])
    print(name, "encoding", "u16" if sim.device_costs.u16 is not None else "f64", f"{ms:.3f} ms/eval",
          {f"seq{k[0]}_ph{k[1]}": (len(v), round(sum(v) / len(v), 4)) for k, v in kinds.items()}, flush=True)
