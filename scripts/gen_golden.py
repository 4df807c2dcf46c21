"""Generate golden vectors from the REFERENCE implementation (fastqaoa).

Run in the dev container only (needs /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python scripts/gen_golden.py

Writes tests/golden/golden.npz.  Every array in it was produced by the
reference's own public API (terms.precompute_cost_vector, qaoa.simulate_qaoa,
statevec.expectation / overlap, distributed.simulate_qaoa_distributed,
distributed.all_to_all_exchange), on seeded inputs restated here so the test
suite can rebuild the same inputs without the reference present.
"""

from __future__ import annotations

import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

from fastqaoa import distributed as D  # noqa: E402
from fastqaoa.mixers import SU2, Mixer  # noqa: E402
from fastqaoa.problems import Graph, cubic_ring_graph, labs_terms, maxcut_terms, triangle_graph  # noqa: E402
from fastqaoa.qaoa import QaoaParams, simulate_qaoa  # noqa: E402
from fastqaoa.statevec import expectation, hamming_weight_state, overlap  # noqa: E402
from fastqaoa.terms import Term, TermPolynomial, compact_costs, precompute_cost_vector  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "golden.npz")

# Pinned random 3-regular graph on 26 vertices (networkx.random_regular_graph(3, 26, seed=1),
# SURVEY.md §8(d) config 2); also committed as tests/golden/maxcut26.edges.
MAXCUT26 = [(0, 4), (0, 18), (0, 22), (1, 7), (1, 18), (1, 21), (2, 4), (2, 11), (2, 25), (3, 12),
            (3, 21), (3, 23), (4, 24), (5, 8), (5, 13), (5, 19), (6, 8), (6, 16), (6, 20), (7, 8),
            (7, 23), (9, 10), (9, 14), (9, 15), (10, 12), (10, 23), (11, 14), (11, 15), (12, 17),
            (13, 19), (13, 24), (14, 16), (15, 18), (16, 25), (17, 20), (17, 22), (19, 22), (20, 25),
            (21, 24)]


def random_poly(seed: int, n: int, max_terms: int | None = None) -> TermPolynomial:
    """Same generator as reference tests/_helpers.py:22-29."""
    rng = np.random.default_rng(seed)
    n_terms = int(rng.integers(1, max_terms or (2 * n + 1)))
    terms = []
    for _ in range(n_terms):
        size = int(rng.integers(0, min(4, n) + 1))
        support = tuple(sorted(rng.choice(n, size=size, replace=False).tolist()))
        terms.append(Term(float(rng.uniform(-2.0, 2.0)), support))
    return TermPolynomial(n, tuple(terms))


def portfolio(n: int, q: float = 0.5, seed: int = 0) -> TermPolynomial:
    """Synthetic mean-variance instance, SURVEY.md §8(d) config 4."""
    rng = np.random.default_rng(seed)
    mu = rng.uniform(0, 1, n)
    A = rng.normal(size=(n, n))
    S = A @ A.T / n
    terms = []
    for i in range(n):
        terms.append(Term(-q * S[i, i] / 2 - q * (S[i].sum() - S[i, i]) / 2 + mu[i] / 2, (i,)))
    for i in range(n):
        for j in range(i + 1, n):
            terms.append(Term(q * S[i, j] / 2, (i, j)))
    terms.append(Term(q * np.trace(S) / 2 + q * (S.sum() - np.trace(S)) / 4 - mu.sum() / 2))
    return TermPolynomial(n, tuple(terms))


def pack_terms(poly: TermPolynomial):
    w = np.array([t.weight for t in poly.terms], dtype=np.float64)
    m = np.array([t.mask for t in poly.terms], dtype=np.int64)
    return w, m


def angles(seed: int, p: int):
    """cli.py:235,246-247 style: rng = default_rng(seed); g, b = U(0,1,p) each."""
    rng = np.random.default_rng(seed)
    return rng.uniform(0, 1, p), rng.uniform(0, 1, p)


def main() -> None:
    g: dict[str, np.ndarray] = {}

    polys = {
        "labs8": labs_terms(8),
        "labs12": labs_terms(12),
        "labs14": labs_terms(14),
        "tri": maxcut_terms(triangle_graph()),
        "cubic12": maxcut_terms(cubic_ring_graph(12)),
        "maxcut26sub14": maxcut_terms(Graph.from_edges(14, [e for e in MAXCUT26 if max(e) < 14])),
        "rand5": random_poly(101, 5),
        "rand8": random_poly(102, 8),
        "rand10": random_poly(103, 10, max_terms=40),
        "port8": portfolio(8),
        "port12": portfolio(12),
    }
    for name, poly in polys.items():
        w, m = pack_terms(poly)
        g[f"terms/{name}/n"] = np.array(poly.n)
        g[f"terms/{name}/w"] = w
        g[f"terms/{name}/m"] = m
        g[f"diag/{name}"] = precompute_cost_vector(poly)

    # compact (uint16) encoding of integer / dyadic diagonals — terms.py:155-175
    for name in ("labs12", "labs14", "cubic12"):
        cc = compact_costs(g[f"diag/{name}"])
        g[f"compact/{name}/values"] = cc.values
        g[f"compact/{name}/scale_offset"] = np.array([cc.scale, cc.offset])

    # full evolutions through the reference's public API
    cases = [
        ("labs8_x_p3", "labs8", "x", 3, None),
        ("labs12_x_p4", "labs12", "x", 4, None),          # BASELINE config 1
        ("labs14_x_p3", "labs14", "x", 3, None),
        ("rand5_x_p2", "rand5", "x", 2, None),
        ("rand10_x_p5", "rand10", "x", 5, None),
        ("cubic12_x_p6", "cubic12", "x", 6, None),
        ("maxcut26sub14_x_p2", "maxcut26sub14", "x", 2, None),
        ("port8_ring_p2", "port8", "xy-ring", 2, 4),
        ("port8_complete_p2", "port8", "xy-complete", 2, 4),
        ("port12_ring_p2", "port12", "xy-ring", 2, 6),
        ("port12_complete_p1", "port12", "xy-complete", 1, 6),
        ("labs8_custom_p2", "labs8", "custom", 2, None),
    ]
    for i, (case, pname, kind, p, hw) in enumerate(cases):
        poly = polys[pname]
        gam, bet = angles(1000 + i, p)
        if kind == "custom":
            mixer = Mixer.custom(lambda b, n=poly.n: [SU2(np.cos(b), np.sin(b))] * n)
        else:
            mixer = Mixer(kind)
        initial = hamming_weight_state(poly.n, hw) if hw is not None else None
        res = simulate_qaoa(poly, QaoaParams(tuple(gam), tuple(bet)), mixer=mixer, initial=initial)
        g[f"sim/{case}/gammas"] = gam
        g[f"sim/{case}/betas"] = bet
        g[f"sim/{case}/state"] = res.state
        g[f"sim/{case}/E"] = np.array(expectation(res.state, res.costs))
        g[f"sim/{case}/overlap"] = np.array(overlap(res.state, res.costs))

    # sharded evolution and the raw exchange — distributed.py:103-122, 280-296
    gam, bet = angles(2000, 3)
    dres = D.simulate_qaoa_distributed(labs_terms(8), QaoaParams(tuple(gam), tuple(bet)), 4)
    g["dist/labs8_K4/gammas"] = gam
    g["dist/labs8_K4/betas"] = bet
    g["dist/labs8_K4/state"] = dres.statevector()
    g["dist/labs8_K4/exchanges"] = np.array(dres.exchange_count)
    rng = np.random.default_rng(2001)
    st = rng.normal(size=64) + 1j * rng.normal(size=64)
    sh = D.scatter(st, 4)
    D.all_to_all_exchange(sh)
    g["exchange/n6K4/in"] = st
    g["exchange/n6K4/out"] = D.gather(sh)

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
