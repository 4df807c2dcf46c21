"""Where the end-to-end time of a synchronous objective evaluation goes
(LABS n=26 p=10 through the public API): per call, CUDA events on the stream
right before / after the call, and the library's own per-pass events
(option time_passes: event 0 right before the first pass).  Prints the GPU
idle time before the first pass (host prologue), the pass span, the tail
(partials sum) and the idle gap between calls (scalar read back + Python)."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_04841_b200 import QaoaSimulator, _lib, labs_terms  # noqa: E402

n, p = int(os.environ.get("N", 26)), 10
rng = np.random.default_rng(0)
g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
sim = QaoaSimulator(terms=labs_terms(n))
for _ in range(3):
    sim.objective(g, b)
torch.cuda.synchronize()
K = 20
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
first, span, tail, gap, walls = [], [], [], [], []
lib = _lib.load()
for mode in ("objective", "simulate+get_expectation"):
    _lib.call("fq_set_option", b"time_passes", 1)
    first.clear(); span.clear(); tail.clear(); gap.clear(); walls.clear()
    t0 = time.perf_counter()
    for i in range(K):
        a, z = evs[i]
        a.record()
        if mode == "objective":
            sim.objective(g + 1e-4 * i, b)
        else:
            sim.get_expectation(sim.simulate_qaoa(g + 1e-4 * i, b))
        z.record()
        z.synchronize()
        cnt = lib.fq_last_passes(None, None, 0)
        # library events: fq_pass_events gives event k (k = 0: before the first pass)
        ms = (ctypes.c_float * 256)()
        info = (ctypes.c_int * (5 * 256))()
        lib.fq_last_passes(info, ms, 256)
        span.append(sum(ms[j] for j in range(cnt)))
        walls.append(a.elapsed_time(z))
    t = (time.perf_counter() - t0) / K
    _lib.call("fq_set_option", b"time_passes", 0)
    gaps = [evs[i][0].elapsed_time(evs[i + 1][0]) - evs[i][0].elapsed_time(evs[i][1]) for i in range(K - 1)]
    print(f"{mode}: host wall {1e3 * t:.3f} ms/eval; call span (events around the call) {np.mean(walls):.3f} ms; "
          f"sum of pass events {np.mean(span):.3f} ms; span - passes {np.mean(walls) - np.mean(span):.3f} ms; "
          f"idle between calls {np.mean(gaps):.3f} ms", flush=True)
# back-to-back device time for comparison
for _ in range(3):
    sim.objective(g, b)
torch.cuda.synchronize()
a, z = evs[0]
a.record()
for i in range(K):
    sim.simulate_qaoa(g, b, reuse_buffer=True)
z.record()
torch.cuda.synchronize()
print(f"back-to-back (no sync): {a.elapsed_time(z) / K:.3f} ms/eval", flush=True)
