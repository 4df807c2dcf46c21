import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2309_04841_b200 import QaoaSimulator, labs_terms, _lib
n, p = 12, 4
rng = np.random.default_rng(0)
g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
sim = QaoaSimulator(terms=labs_terms(n))
for opt in (1, 0):
    _lib.call("fq_set_option", b"res16", opt)
    for _ in range(5): sim.objective(g, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100): sim.simulate_qaoa(g, b, reuse_buffer=True)
    e1.record(); torch.cuda.synchronize()
    print("res16", opt, e0.elapsed_time(e1) / 100, "ms/eval back to back", flush=True)
