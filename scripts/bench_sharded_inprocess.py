"""In-process sharded program vs the single-state program on one B200
(development tool): the same state split into K shard views, so the spanning
(G) passes run over local HBM here — this isolates their on-chip cost from
NVLink, which only a multi-GPU node can measure."""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_04841_b200 import QaoaParams, QaoaSimulator, labs_terms  # noqa: E402
from paper_2309_04841_b200 import distributed as D  # noqa: E402
from paper_2309_04841_b200.qaoa import simulate_qaoa  # noqa: E402


def timed(fn, steps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=27)
    ap.add_argument("--p", type=int, default=10)
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    rng = np.random.default_rng(0)
    params = QaoaParams(tuple(rng.uniform(0, 1, args.p)), tuple(rng.uniform(0, 1, args.p)))
    poly = labs_terms(args.n)
    sim = QaoaSimulator(terms=poly)
    E = {}
    out = {"n": args.n, "p": args.p}
    out["single_ms"] = timed(lambda: E.setdefault("single", simulate_qaoa(poly, params)), args.steps)
    for K in (2, 4, 8):
        out[f"K{K}_ms"] = timed(lambda: D.simulate_qaoa_distributed(poly, params, K), args.steps)
        # the reference's structure: per layer local passes, exchange, k-position pass, exchange
        out[f"K{K}_exchange_ms"] = timed(lambda: D.simulate_qaoa_distributed(poly, params, K, fused=False),
                                         max(1, args.steps // 2))
    r = D.simulate_qaoa_distributed(poly, params, 8)
    out["objective_K8"] = r.expectation()
    out["objective_single"] = sim.get_expectation(sim.simulate_qaoa(params.gammas, params.betas))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
