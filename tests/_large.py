"""Full-size golden cases (tests/golden/golden_large.npz, generated from the
reference by scripts/gen_golden_large.py): problem constructors and the
fingerprint comparison shared by the CPU-oracle and GPU tests."""

import hashlib
import os

import numpy as np

from paper_2309_04841_b200.problems import Graph, labs_terms, maxcut_terms, portfolio_terms

HERE = os.path.dirname(os.path.abspath(__file__))


def maxcut26_edges():
    with open(os.path.join(HERE, "golden", "maxcut26.edges")) as f:
        return [tuple(int(x) for x in line.split()) for line in f if line.strip() and not line.startswith("#")]


# name -> (problem factory, mixer kind, Hamming weight of the initial state or None)
CASES = {
    "labs26_x_p10": (lambda: labs_terms(26), "x", None),
    "labs26_x_p10_ramp": (lambda: labs_terms(26), "x", None),
    "maxcut26_x_p6": (lambda: maxcut_terms(Graph.from_edges(26, maxcut26_edges())), "x", None),
    "labs22_x_p4": (lambda: labs_terms(22), "x", None),
    "port22_ring_p2": (lambda: portfolio_terms(22), "xy-ring", 11),
    "port22_complete_p1": (lambda: portfolio_terms(22), "xy-complete", 11),
    "port26_ring_p1": (lambda: portfolio_terms(26), "xy-ring", 13),
    "labs30_x_p3": (lambda: labs_terms(30), "x", None),  # BASELINE config 3's size, the reference's n <= 30 limit
    "port26_complete_p1": (lambda: portfolio_terms(26), "xy-complete", 13),  # BASELINE config 4, full size
    "port26_ring_p2": (lambda: portfolio_terms(26), "xy-ring", 13),
    "labs30_x_p10": (lambda: labs_terms(30), "x", None),  # BASELINE config 3 at its full depth
}


def diag_sha256(costs: np.ndarray) -> np.ndarray:
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(costs, dtype=np.float64).tobytes()).digest(),
                         dtype=np.uint8)


def check_fingerprint(g, name, costs, state, E, overlap, atol=1e-10, rtol=1e-10):
    """Bit-exact diagonal; E / overlap to rtol; sampled amplitudes and the
    1024 block norms to atol (fp64 north-star tolerance)."""
    np.testing.assert_array_equal(diag_sha256(costs), g[f"{name}/diag_sha256"])
    e_ref = float(g[f"{name}/E"])
    assert abs(E - e_ref) <= rtol * max(1.0, abs(e_ref)), (E, e_ref)
    assert abs(overlap - float(g[f"{name}/overlap"])) <= atol, (overlap, float(g[f"{name}/overlap"]))
    idx = g[f"{name}/idx"]
    np.testing.assert_allclose(state[idx], g[f"{name}/amp"], rtol=0, atol=atol)
    blocks = (np.abs(state) ** 2).reshape(1024, -1).sum(axis=1)
    np.testing.assert_allclose(blocks, g[f"{name}/block_norm2"], rtol=0, atol=atol)
