"""Host-overhead breakdown of one small-n objective() call (config 1)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_04841_b200 import QaoaSimulator, _lib, labs_terms  # noqa: E402

sim = QaoaSimulator(terms=labs_terms(12))
rng = np.random.default_rng(0)
g, b = rng.uniform(0, 1, 4), rng.uniform(0, 1, 4)
sim.objective(g, b)
og = sim._graph_ctx[1]


def t(fn, reps=3000):
    for _ in range(100):
        fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e6


st = _lib.stream()
lib = _lib.load()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
print(f"objective(): {t(lambda: sim.objective(g, b)):.1f} us")
print(f"graph run (ctypes + launch + sync): {t(og.run):.1f} us")
print(f"stream sync alone: {t(torch.cuda.synchronize):.1f} us")
print(f"ctypes call of fq_set_option: {t(lambda: lib.fq_set_option(b'fuse', 1)):.1f} us")
print(f"_lib.stream(): {t(_lib.stream):.1f} us")
ev0.record()
for _ in range(200):
    og.run()
ev1.record()
torch.cuda.synchronize()
print(f"events around 200 runs: {ev0.elapsed_time(ev1) / 200 * 1e3:.1f} us per run")
