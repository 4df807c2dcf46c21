"""XY-mixer layer timing (BASELINE config 4: portfolio n=26, Hamming weight
13, float64 costs): device time per layer of the tiled XY program, evolved in
place on a resident state (no initial-state copy), complex128 and complex64,
and complex128 with gamma = 0 (no phase: the phase share of a layer)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_04841_b200 import QaoaSimulator, _lib, hamming_weight_state  # noqa: E402
from paper_2309_04841_b200.mixers import run_program  # noqa: E402
from paper_2309_04841_b200.problems import portfolio_terms  # noqa: E402

n = int(os.environ.get("N", 26))
p = int(os.environ.get("P", 4))
only = os.environ.get("ONLY", "")
poly = portfolio_terms(n)
sim = QaoaSimulator(terms=poly)
dc = sim.device_costs
init = torch.from_numpy(hamming_weight_state(n, n // 2)).cuda()
rng = np.random.default_rng(0)
g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
for kind in ("xy-ring", "xy-complete"):
    if only and only != kind:
        continue
    for dt, gam in ((torch.complex128, g), (torch.complex64, g), (torch.complex128, 0 * g)):
        state = init.to(dt).clone()
        e = torch.empty(1, dtype=torch.float64, device="cuda")
        layers = [(float(x), float(y), 1, 0, n) for x, y in zip(gam, b)]
        fn = lambda: run_program(state, n, kind, layers, dc=dc, expectation_out=e)  # noqa: E731
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(json.dumps({"mixer": kind, "dtype": str(dt).split(".")[-1], "n": n, "p": p,
                          "phase": bool(np.any(gam)),
                          "ms_per_layer": ms / p, "ms_program": ms,
                          "norm": float(torch.linalg.vector_norm(state).item())}), flush=True)
        del state
