"""In-process sharding (K logical workers on one GPU): parity with the
single-node evolution, the reference's golden sharded run, exchange-count
contract (reference tests/test_distributed.py)."""

import numpy as np
import pytest

from _helpers import random_pairs, random_state, random_su2_coeffs
from oracle import oracle as O
from paper_2309_04841_b200 import SU2, QaoaParams, TermPolynomial, hamming_weight_state, labs_terms, simulate_qaoa
from paper_2309_04841_b200 import distributed as D

pytestmark = pytest.mark.gpu


def test_exchange_golden_and_involution(golden):
    sh = D.scatter(golden["exchange/n6K4/in"], 4)
    D.all_to_all_exchange(sh)
    np.testing.assert_array_equal(D.gather(sh), golden["exchange/n6K4/out"])
    D.all_to_all_exchange(sh)
    np.testing.assert_array_equal(D.gather(sh), golden["exchange/n6K4/in"])
    assert sh.exchange_count == 2


@pytest.mark.parametrize("n,K", [(4, 4), (5, 2), (6, 4), (8, 8), (16, 4)])
def test_exchange_matches_transpose_oracle(n, K):
    rng = np.random.default_rng(22 + n)
    x = random_state(rng, n)
    sh = D.scatter(x, K)
    D.all_to_all_exchange(sh)
    np.testing.assert_array_equal(D.gather(sh), O.transpose_oracle(x, sh.k))


def test_split_validation():
    with pytest.raises(ValueError, match="power of two"):
        D.scatter(np.ones(16, dtype=complex) / 4, 3)
    with pytest.raises(ValueError, match="subchunks"):
        D.scatter(np.ones(8, dtype=complex), 4)
    with pytest.raises(ValueError, match="subchunks"):
        D.simulate_qaoa_distributed(labs_terms(3), QaoaParams((), ()), 4)


@pytest.mark.parametrize("n,K", [(4, 4), (6, 4), (6, 2), (7, 2), (10, 4), (15, 2), (16, 4)])
def test_uniform_su2_distributed_matches_single_node(n, K):
    rng = np.random.default_rng(24 + n + K)
    us = [SU2(*random_su2_coeffs(rng)) for _ in range(n)]
    x = random_state(rng, n)
    ref = x.copy()
    O.apply_uniform_su2(ref, [(u.a, u.b) for u in us])
    sh = D.scatter(x, K)
    D.apply_uniform_su2_distributed(sh, us)
    np.testing.assert_allclose(D.gather(sh), ref, atol=1e-12)
    assert sh.exchange_count == 2


@pytest.mark.parametrize("n,K", [(6, 2), (6, 4), (5, 2), (8, 4)])
def test_xy_every_pair_matches_single_node(n, K):
    rng = np.random.default_rng(26 + n + K)
    beta = 0.44
    for i in range(n):
        for j in range(i + 1, n):
            x = random_state(rng, n)
            ref = x.copy()
            O.apply_xy(ref, beta, i, j)
            sh = D.scatter(x, K)
            D.apply_xy_distributed(sh, beta, i, j)
            np.testing.assert_allclose(D.gather(sh), ref, atol=1e-12, err_msg=f"pair ({i},{j})")
    sh = D.scatter(random_state(rng, 4), 4)
    with pytest.raises(ValueError, match="spans"):
        D.apply_xy_distributed(sh, 0.3, 1, 2)


def test_labs8_matches_reference_sharded_run(golden):
    g, b = golden["dist/labs8_K4/gammas"], golden["dist/labs8_K4/betas"]
    res = D.simulate_qaoa_distributed(labs_terms(8), QaoaParams(tuple(g), tuple(b)), 4)
    np.testing.assert_allclose(res.statevector(), golden["dist/labs8_K4/state"], atol=1e-11)
    assert res.exchange_count == int(golden["dist/labs8_K4/exchanges"])


@pytest.mark.parametrize("n,K,p", [(8, 4, 3), (6, 2, 2), (16, 4, 3), (18, 8, 2), (14, 2, 5)])
def test_labs_sharded_vs_single(n, K, p):
    rng = np.random.default_rng(29 + n)
    params = QaoaParams(tuple(rng.uniform(-1, 1, p)), tuple(rng.uniform(-1, 1, p)))
    single = simulate_qaoa(labs_terms(n), params)
    dist = D.simulate_qaoa_distributed(labs_terms(n), params, K)
    np.testing.assert_allclose(dist.statevector(), single.state, atol=1e-11 * np.abs(single.state).max() * 2 ** (n / 2))
    assert dist.exchange_count == 2 * p
    assert dist.expectation() == pytest.approx(float(single._expectation_dev.item()), rel=1e-10)


def test_xy_ring_sharded_and_observables():
    rng = np.random.default_rng(30)
    n = 6
    poly = labs_terms(n)
    init = hamming_weight_state(n, 3)
    params = QaoaParams(tuple(rng.uniform(-1, 1, 2)), tuple(rng.uniform(-1, 1, 2)))
    single = simulate_qaoa(poly, params, mixer="xy-ring", initial=init)
    dist = D.simulate_qaoa_distributed(poly, params, 4, mixer="xy-ring", initial=init)
    np.testing.assert_allclose(dist.statevector(), single.state, atol=1e-11)
    rng = np.random.default_rng(31)
    n, K = 7, 2
    pairs = random_pairs(rng, n)
    costs = O.precompute_cost_vector(n, pairs)
    x = random_state(rng, n)
    sh = D.scatter(x, K)
    sc = D.shard_costs(costs, K)
    assert D.expectation_distributed(sh, sc) == pytest.approx(O.expectation(x, costs), abs=1e-12)
    assert D.overlap_distributed(sh, sc) == pytest.approx(O.overlap(x, costs), abs=1e-12)
    res = D.simulate_qaoa_distributed(labs_terms(4), QaoaParams((0.2,), (0.4,)), 2)
    single = simulate_qaoa(labs_terms(4), QaoaParams((0.2,), (0.4,)))
    np.testing.assert_allclose(res.to_result().state, single.state, atol=1e-12)
    np.testing.assert_array_equal(res.to_result().costs, single.costs)


def test_single_worker_equals_single_node():
    rng = np.random.default_rng(28)
    poly = TermPolynomial.from_pairs(5, random_pairs(rng, 5))
    params = QaoaParams(tuple(rng.uniform(-1, 1, 2)), tuple(rng.uniform(-1, 1, 2)))
    np.testing.assert_allclose(D.simulate_qaoa_distributed(poly, params, 1).statevector(),
                               simulate_qaoa(poly, params).state, atol=1e-13)


@pytest.mark.parametrize("n,K,p", [(10, 2, 2), (14, 4, 3), (17, 8, 2), (20, 16, 1)])
def test_fused_global_pass_equals_exchange_path(n, K, p):
    """The peer-memory global-qubit pass (fq_global_su2_pass) replaces Alg. 4's
    exchange -> k-position pass -> exchange with identical results and the same
    logical exchange count."""
    from paper_2309_04841_b200.distributed import simulate_qaoa_distributed

    rng = np.random.default_rng(n + K)
    g, b = rng.uniform(0, 1, p), rng.uniform(-1.5, 1.5, p)
    params = QaoaParams(tuple(g), tuple(b))
    a = simulate_qaoa_distributed(labs_terms(n), params, K, fused=True)
    r = simulate_qaoa_distributed(labs_terms(n), params, K, fused=False)
    np.testing.assert_allclose(a.statevector(), r.statevector(), rtol=0, atol=1e-12)
    assert a.exchange_count == r.exchange_count == 2 * p


@pytest.mark.parametrize("n,K", [(9, 2), (12, 4), (15, 8)])
def test_fused_global_pass_custom_mixer(n, K):
    """Custom per-qubit SU(2) mixers: peer-memory global pass == exchange path."""
    from paper_2309_04841_b200 import Mixer
    from paper_2309_04841_b200.distributed import simulate_qaoa_distributed

    rng = np.random.default_rng(n)
    tabs = {}

    def factory(beta):
        if beta not in tabs:
            tabs[beta] = [SU2(*random_su2_coeffs(rng)) for _ in range(n)]
        return tabs[beta]

    params = QaoaParams(tuple(rng.uniform(0, 1, 2)), (0.3, 0.7))
    mixer = Mixer.custom(factory)
    a = simulate_qaoa_distributed(labs_terms(n), params, K, mixer=mixer, fused=True)
    r = simulate_qaoa_distributed(labs_terms(n), params, K, mixer=mixer, fused=False)
    np.testing.assert_allclose(a.statevector(), r.statevector(), rtol=0, atol=1e-12)
    assert a.exchange_count == r.exchange_count == 4
