"""Shared seeded generators (same distributions as reference tests/_helpers.py:9-41)."""

import numpy as np


def random_su2_coeffs(rng):
    theta, phi_a, phi_b = rng.uniform(0.0, 2.0 * np.pi, 3)
    return complex(np.cos(theta) * np.exp(1j * phi_a)), complex(np.sin(theta) * np.exp(1j * phi_b))


def random_state(rng, n):
    state = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return state / np.linalg.norm(state)


def random_pairs(rng, n, max_terms=None, integer=False):
    """(weight, support) pairs: float U(-2,2) weights (or small integers)."""
    n_terms = int(rng.integers(1, max_terms or (2 * n + 1)))
    out = []
    for _ in range(n_terms):
        size = int(rng.integers(0, min(4, n) + 1))
        support = tuple(sorted(rng.choice(n, size=size, replace=False).tolist()))
        w = float(rng.integers(-3, 4)) if integer else float(rng.uniform(-2.0, 2.0))
        out.append((w, support))
    return out


def golden_terms(g, name):
    w = g[f"terms/{name}/w"]
    m = g[f"terms/{name}/m"]
    n = int(g[f"terms/{name}/n"])
    pairs = [(float(wi), tuple(b for b in range(n) if (int(mi) >> b) & 1)) for wi, mi in zip(w, m)]
    return n, pairs
