"""fq_qaoa_evolve_sharded in the in-process worker model (all K shard views
on one device, one stream): one plan over all n qubits, local groups as
passes on every shard, the global group as passes whose tiles span the K
shards (the kernels a multi-GPU rank runs over peer memory).  Compared
against the single-GPU program and the oracle."""

import numpy as np
import pytest

from _helpers import random_pairs, random_state, random_su2_coeffs
from oracle import oracle as O
from paper_2309_04841_b200 import SU2, Mixer, QaoaParams, TermPolynomial, simulate_qaoa
from paper_2309_04841_b200 import distributed as D
from paper_2309_04841_b200.problems import labs_terms

pytestmark = pytest.mark.gpu


def _params(rng, p, zero_gamma=False):
    g = rng.uniform(-1, 1, p)
    if zero_gamma and p > 1:
        g[1] = 0.0
    return QaoaParams(tuple(g), tuple(rng.uniform(-1.6, 1.6, p)))


@pytest.mark.parametrize("n,K,p", [(13, 2, 1), (14, 4, 3), (15, 8, 2), (17, 2, 4), (20, 4, 5), (23, 8, 3),
                                   (25, 2, 2), (27, 8, 2)])
def test_sharded_program_matches_single_gpu(n, K, p):
    rng = np.random.default_rng(100 + n + K)
    params = _params(rng, p, zero_gamma=True)
    poly = labs_terms(n)
    single = simulate_qaoa(poly, params)
    res = D.simulate_qaoa_distributed(poly, params, K)
    ref = single.state
    # 1e-10 relative to the largest amplitude (amplitudes are ~2^-n/2)
    np.testing.assert_allclose(res.statevector(), ref, rtol=0, atol=1e-10 * np.abs(ref).max())
    assert res.exchange_count == 2 * p
    assert res.expectation() == pytest.approx(float(single._expectation_dev.item()), rel=1e-10)


@pytest.mark.parametrize("n,K", [(14, 2), (16, 4), (18, 8)])
def test_sharded_float_costs_and_initial_state(n, K):
    """float64 costs (sincos phase in the spanning passes) and an explicit initial state."""
    rng = np.random.default_rng(7 * n + K)
    poly = TermPolynomial.from_pairs(n, random_pairs(rng, n, max_terms=3 * n))
    params = _params(rng, 3)
    init = random_state(rng, n)
    res = D.simulate_qaoa_distributed(poly, params, K, initial=init)
    costs = res.to_result().costs
    ref = O.simulate(costs, params.gammas, params.betas, "x", init)
    np.testing.assert_allclose(res.statevector(), ref, rtol=0, atol=1e-12)
    assert res.expectation() == pytest.approx(O.expectation(ref, costs), rel=1e-10, abs=1e-12)


@pytest.mark.parametrize("n,K", [(13, 2), (16, 8)])
def test_sharded_custom_mixer_vs_oracle(n, K):
    rng = np.random.default_rng(n * K)
    tabs = {}

    def factory(beta):
        if beta not in tabs:
            tabs[beta] = [SU2(*random_su2_coeffs(rng)) for _ in range(n)]
        return tabs[beta]

    params = QaoaParams((0.3, -0.2, 0.5), (0.3, 0.7, -0.4))
    mixer = Mixer.custom(factory)
    res = D.simulate_qaoa_distributed(labs_terms(n), params, K, mixer=mixer)
    single = simulate_qaoa(labs_terms(n), params, mixer=mixer)
    np.testing.assert_allclose(res.statevector(), single.state, rtol=0, atol=1e-12)


def test_sharded_zero_layers():
    res = D.simulate_qaoa_distributed(labs_terms(14), QaoaParams((), ()), 4)
    np.testing.assert_allclose(res.statevector(), np.full(1 << 14, 2 ** -7), rtol=0, atol=1e-15)


@pytest.mark.parametrize("kind,n,K,p", [("xy-ring", 14, 2, 2), ("xy-ring", 17, 8, 3), ("xy-complete", 14, 4, 1),
                                        ("xy-complete", 16, 8, 2), ("xy-complete", 15, 2, 2)])
def test_sharded_xy_matches_single_gpu(kind, n, K, p):
    """XY mixers: the tiled XY plan over all n qubits; passes holding global
    qubits span the shards they cover (replaces park-and-exchange per global pair)."""
    from paper_2309_04841_b200 import hamming_weight_state
    from paper_2309_04841_b200.problems import portfolio_terms

    rng = np.random.default_rng(3 * n + K)
    params = _params(rng, p)
    poly = portfolio_terms(n)
    init = hamming_weight_state(n, n // 2)
    single = simulate_qaoa(poly, params, mixer=kind, initial=init)
    res = D.simulate_qaoa_distributed(poly, params, K, mixer=kind, initial=init)
    np.testing.assert_allclose(res.statevector(), single.state, rtol=0, atol=1e-12)
    assert res.expectation() == pytest.approx(float(single._expectation_dev.item()), rel=1e-10, abs=1e-12)


def test_sharded_xy_exchange_count_matches_reference_path():
    from paper_2309_04841_b200 import hamming_weight_state
    from paper_2309_04841_b200.problems import portfolio_terms

    n, K = 14, 4
    params = QaoaParams((0.2,), (0.4,))
    init = hamming_weight_state(n, 7)
    a = D.simulate_qaoa_distributed(portfolio_terms(n), params, K, mixer="xy-ring", initial=init)
    r = D.simulate_qaoa_distributed(portfolio_terms(n), params, K, mixer="xy-ring", initial=init, fused=False)
    assert a.exchange_count == r.exchange_count
    np.testing.assert_allclose(a.statevector(), r.statevector(), rtol=0, atol=1e-12)
