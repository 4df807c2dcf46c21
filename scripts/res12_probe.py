"""Config 1 (LABS n=12 p=4) probe: device time of one evaluation back to back,
and batched throughput (k_resident8)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_04841_b200 import QaoaSimulator, _lib, labs_terms  # noqa: E402

n, p = 12, 4
rng = np.random.default_rng(0)
g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
sim = QaoaSimulator(terms=labs_terms(n))
B = 4096
G, Bt = rng.uniform(0, 1, (B, p)), rng.uniform(0, 1, (B, p))


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for _ in range(200):  # clocks up before the first timed variant
    sim.simulate_qaoa_batched(G, Bt)
for rep in range(2):
    ms1 = timed(lambda: sim.simulate_qaoa(g, b, reuse_buffer=True), 200)
    msb = timed(lambda: sim.simulate_qaoa_batched(G, Bt), 10)
    print(f"rep {rep}: {ms1 * 1e3:.1f} us/eval back to back; batched {B} sets: {msb:.3f} ms "
          f"= {B / msb * 1e3 / 1e6:.2f} M evals/s", flush=True)
