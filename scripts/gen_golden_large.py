"""Full-size golden pins from the REFERENCE implementation (fastqaoa).

Run in the dev container only (needs /root/reference; ~5 min on 8 cores):

    NUMBA_CACHE_DIR=/tmp/numba_cache python scripts/gen_golden_large.py [case ...]

The BASELINE configurations are too large to commit as state dumps (1 GiB
per n=26 state), so each case stores size-independent fingerprints of the
reference's own outputs, all produced through its public API
(terms.precompute_cost_vector, qaoa.simulate_qaoa, statevec.expectation /
overlap):

* ``diag_sha256``   — SHA-256 of the float64 cost diagonal's bytes (bit-exact pin);
* ``E``, ``overlap`` — the objective and ground-state overlap;
* ``idx``/``amp``   — 4096 amplitudes at seeded random indices;
* ``block_norm2``   — sum |psi|^2 over each of 1024 contiguous blocks
                       (a checksum of checksums over the whole state).

Writes tests/golden/golden_large.npz (merged with any cases already there).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from fastqaoa.mixers import Mixer  # noqa: E402
from fastqaoa.problems import Graph, labs_terms, maxcut_terms  # noqa: E402
from fastqaoa.qaoa import QaoaParams, QaoaSimulator  # noqa: E402
from fastqaoa.statevec import hamming_weight_state  # noqa: E402
from gen_golden import MAXCUT26, portfolio  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "golden_large.npz")
N_SAMPLES = 4096
N_BLOCKS = 1024


def bench_angles(p: int):
    """bench.py / cli.py:235,246-247: default_rng(0), gammas then betas U(0,1)."""
    rng = np.random.default_rng(0)
    return rng.uniform(0, 1, p), rng.uniform(0, 1, p)


def ramp_angles(p: int):
    """Linear-ramp schedule: gamma 0.01 -> 0.1, beta 0.6 -> 0.06."""
    return np.linspace(0.01, 0.1, p), np.linspace(0.6, 0.06, p)


CASES = {
    # name: (problem factory, mixer, p, angle schedule, Hamming weight of the initial state)
    "labs26_x_p10": (lambda: labs_terms(26), "x", 10, bench_angles, None),
    "labs26_x_p10_ramp": (lambda: labs_terms(26), "x", 10, ramp_angles, None),
    "maxcut26_x_p6": (lambda: maxcut_terms(Graph.from_edges(26, MAXCUT26)), "x", 6, bench_angles, None),
    "labs22_x_p4": (lambda: labs_terms(22), "x", 4, bench_angles, None),
    "port22_ring_p2": (lambda: portfolio(22), "xy-ring", 2, bench_angles, 11),
    "port22_complete_p1": (lambda: portfolio(22), "xy-complete", 1, bench_angles, 11),
    "port26_ring_p1": (lambda: portfolio(26), "xy-ring", 1, bench_angles, 13),
    # BASELINE config 3's size (the reference's n <= 30 limit): ~15 min on 8 cores, mostly precompute
    "labs30_x_p3": (lambda: labs_terms(30), "x", 3, bench_angles, None),
    # BASELINE config 4 at full size: XY-complete n=26 (325 gates per layer) and XY-ring at p=2
    "port26_complete_p1": (lambda: portfolio(26), "xy-complete", 1, bench_angles, 13),
    "port26_ring_p2": (lambda: portfolio(26), "xy-ring", 2, bench_angles, 13),
    # BASELINE config 3 at its full depth (LABS n=30, p=10): ~25 min on 8 cores
    "labs30_x_p10": (lambda: labs_terms(30), "x", 10, bench_angles, None),
}


def fingerprint(state: np.ndarray, costs: np.ndarray, seed: int) -> dict:
    n = state.size.bit_length() - 1
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(state.size, size=min(N_SAMPLES, state.size), replace=False)).astype(np.int64)
    blocks = (np.abs(state) ** 2).reshape(N_BLOCKS, -1).sum(axis=1)
    return {"n": np.array(n), "idx": idx, "amp": state[idx].copy(), "block_norm2": blocks}


def main(names) -> None:
    g = dict(np.load(OUT)) if os.path.exists(OUT) else {}
    for ci, name in enumerate(names):
        make, kind, p, sched, hw = CASES[name]
        poly = make()
        t0 = time.perf_counter()
        sim = QaoaSimulator(terms=poly, mixer=Mixer(kind))
        costs = sim.get_cost_diagonal()
        t_pre = time.perf_counter() - t0
        gam, bet = sched(p)
        initial = hamming_weight_state(poly.n, hw) if hw is not None else None
        t0 = time.perf_counter()
        res = sim.simulate_qaoa(tuple(gam), tuple(bet), initial=initial)
        E = sim.get_expectation(res)
        ov = sim.get_overlap(res)
        t_sim = time.perf_counter() - t0
        g[f"{name}/gammas"] = np.asarray(gam, dtype=np.float64)
        g[f"{name}/betas"] = np.asarray(bet, dtype=np.float64)
        g[f"{name}/diag_sha256"] = np.frombuffer(hashlib.sha256(np.ascontiguousarray(costs).tobytes()).digest(),
                                                 dtype=np.uint8)
        g[f"{name}/diag_minmax"] = np.array([costs.min(), costs.max()])
        g[f"{name}/E"] = np.array(E)
        g[f"{name}/overlap"] = np.array(ov)
        for k, v in fingerprint(res.state, costs, 9000 + sum(map(ord, name))).items():
            g[f"{name}/{k}"] = v
        print(f"{name}: precompute {t_pre:.1f}s, simulate+observables {t_sim:.1f}s, E={E!r}", flush=True)
        del res, sim, costs
        np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
