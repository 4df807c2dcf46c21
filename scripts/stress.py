"""Randomised stress run (development tool): random problems, depths, angles,
mixers, state types and shardings against the CPU oracle, for a time budget.
Prints every failure with its seed; exits 1 if any."""

import os
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from _helpers import random_pairs, random_state, random_su2_coeffs  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2309_04841_b200 import SU2, Mixer, QaoaParams, QaoaSimulator, TermPolynomial, hamming_weight_state  # noqa: E402
from paper_2309_04841_b200.distributed import simulate_qaoa_distributed  # noqa: E402


def one(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(13, 23))  # n = 21: 12 + 9-target groups (lane butterflies)
    p = int(rng.integers(0, 5))
    kind = ["x", "x", "custom", "xy-ring", "xy-complete"][int(rng.integers(0, 5))]
    if kind == "xy-complete":
        n = min(n, 16)
    c64 = rng.random() < 0.3
    integer = rng.random() < 0.6
    poly = TermPolynomial.from_pairs(n, random_pairs(rng, n, max_terms=3 * n, integer=integer))
    g = rng.uniform(-2, 2, p)
    if p and rng.random() < 0.3:
        g[int(rng.integers(0, p))] = 0.0
    b = rng.uniform(-2, 2, p)
    tabs = {}

    def factory(beta):
        if beta not in tabs:
            tabs[beta] = [SU2(*random_su2_coeffs(rng)) for _ in range(n)]
        return tabs[beta]

    mixer = Mixer.custom(factory) if kind == "custom" else Mixer(kind)
    init = None
    if kind.startswith("xy"):
        init = hamming_weight_state(n, int(rng.integers(0, n + 1))) if rng.random() < 0.6 else random_state(rng, n)
    elif rng.random() < 0.2:
        init = random_state(rng, n)
    K = 1 << int(rng.integers(0, 4))
    if n - (K.bit_length() - 1) < 12:
        K = 1
    if c64 and kind == "custom" and K > 1:
        K = 1
    dtype = "complex64" if c64 else None
    if K > 1:
        res = simulate_qaoa_distributed(poly, QaoaParams(tuple(g), tuple(b)), K, mixer=mixer, initial=init, dtype=dtype)
        state = res.statevector()
        costs = res.costs
        E = res.expectation()
    else:
        sim = QaoaSimulator(terms=poly, mixer=mixer, dtype=dtype)
        r = sim.simulate_qaoa(g, b, initial=init)
        state = sim.get_statevector(r)
        costs = sim.get_cost_diagonal()
        E = sim.get_expectation(r)
    su2f = (lambda beta: [(u.a, u.b) for u in factory(beta)]) if kind == "custom" else None
    ref = O.simulate(costs, g, b, kind, init, su2_factory=su2f)
    tol = 1e-4 * max(np.abs(ref).max(), 1e-30) if c64 else 1e-11
    err = np.abs(state.astype(np.complex128) - ref).max()
    e_ref = O.expectation(ref, costs)
    e_tol = (1e-4 * max(abs(e_ref), np.abs(costs).max())) if c64 else 1e-9 * max(1.0, abs(e_ref))
    ok = err <= tol and abs(E - e_ref) <= e_tol
    return ok, dict(n=n, p=p, kind=kind, c64=c64, K=K, integer=integer, init=init is not None, err=err, dE=abs(E - e_ref))


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    t0 = time.time()
    seed, fails, runs = 1000, 0, 0
    while time.time() - t0 < budget:
        seed += 1
        try:
            ok, info = one(seed)
        except Exception:  # noqa: BLE001
            ok, info = False, {"exception": traceback.format_exc(limit=3)}
        runs += 1
        if not ok:
            fails += 1
            if fails <= 20:
                print("FAIL seed", seed, info, flush=True)
    print(f"stress: {runs} random programs, {fails} failures, {time.time() - t0:.0f} s", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
