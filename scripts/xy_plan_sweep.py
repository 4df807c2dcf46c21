"""Measure every XY-complete pass-cut candidate the planner prices (option
xy_row_cap x xy_min_run) at n = 26: passes, register rounds and device ms per
layer, to check the cost model's choice against the hardware."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_04841_b200 import QaoaSimulator, _lib, hamming_weight_state  # noqa: E402
from paper_2309_04841_b200.mixers import run_program  # noqa: E402
from paper_2309_04841_b200.problems import portfolio_terms  # noqa: E402

n, p = 26, 2
kind = os.environ.get("KIND", "xy-complete")
sim = QaoaSimulator(terms=portfolio_terms(n))
dc = sim.device_costs
init = torch.from_numpy(hamming_weight_state(n, n // 2)).cuda()
rng = np.random.default_rng(0)
g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
layers = [(float(x), float(y), 1, 0, n) for x, y in zip(g, b)]
for cap in (0, 1, 2, 3, 4, 6, 64):
    for mr in (0, 3, 4, 5):
        if (cap == 0) != (mr == 0):
            continue
        _lib.call("fq_set_option", b"xy_row_cap", cap)
        _lib.call("fq_set_option", b"xy_min_run", mr)
        rounds = ctypes.c_int()
        passes = _lib.load().fq_plan_xy_passes(n, _lib.MIXER_CODES[kind], ctypes.byref(rounds))
        state = init.clone()
        e = torch.empty(1, dtype=torch.float64, device="cuda")
        fn = lambda: run_program(state, n, kind, layers, dc=dc, expectation_out=e)  # noqa: E731
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"row_cap": cap, "min_run": mr, "passes": passes, "rounds": rounds.value,
                          "ms_per_layer": e0.elapsed_time(e1) / 3 / p}), flush=True)
_lib.call("fq_set_option", b"xy_row_cap", 0)
_lib.call("fq_set_option", b"xy_min_run", 0)
