"""Property-based parity (hypothesis, derandomised profile of tests/conftest.py,
as the reference's own tests/conftest.py:6-9): random problem sizes across
the resident (n <= 12) and tiled (n >= 13) paths, random depths, angles,
mixers, term lists and initial states, every result against the CPU oracle;
plus the invariants the reference tests pin (norm, Hamming-weight
conservation of XY mixers, gamma = 0 identity, E within [min c, max c])."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from _helpers import random_pairs, random_state
from oracle import oracle as O
from paper_2309_04841_b200 import Mixer, QaoaSimulator, TermPolynomial, hamming_weight_state

pytestmark = pytest.mark.gpu

KINDS = ["x", "xy-ring", "xy-complete"]


@settings(max_examples=40, deadline=None)
@given(n=st.integers(2, 17), p=st.integers(0, 4), kind=st.sampled_from(KINDS), seed=st.integers(0, 2**31 - 1),
       integer=st.booleans())
def test_random_programs_match_oracle(n, p, kind, seed, integer):
    rng = np.random.default_rng(seed)
    g = rng.uniform(-2, 2, p)
    b = rng.uniform(-2, 2, p)
    if p and rng.random() < 0.3:
        g[rng.integers(0, p)] = 0.0  # gamma = 0 layers take the identity path (statevec.py:76-77)
    poly = TermPolynomial.from_pairs(n, random_pairs(rng, n, max_terms=3 * n, integer=integer))
    sim = QaoaSimulator(terms=poly, mixer=Mixer(kind))
    init = None
    if kind != "x":
        w = int(rng.integers(0, n + 1))
        init = hamming_weight_state(n, w) if rng.random() < 0.5 else random_state(rng, n)
    res = sim.simulate_qaoa(g, b, initial=init)
    costs = sim.get_cost_diagonal()
    np.testing.assert_array_equal(costs, O.precompute_cost_vector(n, [(t.weight, t.support) for t in poly.terms]))
    ref = O.simulate(costs, g, b, kind, None if init is None else np.array(init))
    np.testing.assert_allclose(res.state, ref, rtol=0, atol=1e-11)
    E = sim.get_expectation(res)
    assert E == pytest.approx(O.expectation(ref, costs), rel=1e-10, abs=1e-10)
    assert costs.min() - 1e-9 <= E <= costs.max() + 1e-9
    assert np.sum(np.abs(res.state) ** 2) == pytest.approx(1.0, abs=1e-11)


@settings(max_examples=25, deadline=None)
@given(n=st.integers(13, 18), kind=st.sampled_from(["xy-ring", "xy-complete"]), w=st.integers(0, 18),
       seed=st.integers(0, 2**31 - 1))
def test_xy_conserves_hamming_weight(n, kind, w, seed):
    w = min(w, n)
    rng = np.random.default_rng(seed)
    poly = TermPolynomial.from_pairs(n, random_pairs(rng, n))
    sim = QaoaSimulator(terms=poly, mixer=kind)
    res = sim.simulate_qaoa(rng.uniform(-1, 1, 2), rng.uniform(-2, 2, 2), initial=hamming_weight_state(n, w))
    pop = np.bitwise_count(np.arange(1 << n, dtype=np.uint64))
    assert np.sum(np.abs(res.state[pop != w]) ** 2) < 1e-24
    assert np.sum(np.abs(res.state[pop == w]) ** 2) == pytest.approx(1.0, abs=1e-11)


@settings(max_examples=20, deadline=None)
@given(n=st.integers(13, 17), k=st.integers(1, 3), p=st.integers(0, 4), seed=st.integers(0, 2**31 - 1),
       integer=st.booleans())
def test_random_sharded_programs_match_single_gpu(n, k, p, seed, integer):
    """fq_qaoa_evolve_sharded (in-process, K shard views) == the single-state program."""
    from paper_2309_04841_b200 import QaoaParams
    from paper_2309_04841_b200.distributed import simulate_qaoa_distributed
    from paper_2309_04841_b200.qaoa import simulate_qaoa

    if n - k < 12:
        k = n - 12
    rng = np.random.default_rng(seed)
    poly = TermPolynomial.from_pairs(n, random_pairs(rng, n, max_terms=3 * n, integer=integer))
    g = rng.uniform(-2, 2, p)
    if p and rng.random() < 0.3:
        g[rng.integers(0, p)] = 0.0
    params = QaoaParams(tuple(g), tuple(rng.uniform(-2, 2, p)))
    init = random_state(rng, n) if rng.random() < 0.3 else None
    single = simulate_qaoa(poly, params, initial=init)
    res = simulate_qaoa_distributed(poly, params, 1 << k, initial=init)
    np.testing.assert_allclose(res.statevector(), single.state, rtol=0, atol=1e-12)
    assert res.expectation() == pytest.approx(float(single._expectation_dev.item()), rel=1e-10, abs=1e-10)
