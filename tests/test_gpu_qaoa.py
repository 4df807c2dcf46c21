"""Simulator-level parity: the fused evolution (resident n <= 12, tiled
passes n >= 13, float64 and uint16 cost paths, X / custom / XY mixers)
against the reference's golden states and the CPU oracle; plus the
reference's API contract (tests/test_qaoa.py, test_statevec.py,
test_mixers.py).  Tolerance: amplitudes 1e-10 absolute (fp64, north star),
objectives 1e-10 relative."""

import numpy as np
import pytest
import torch

from _helpers import golden_terms, random_pairs, random_state, random_su2_coeffs
from oracle import oracle as O
from paper_2309_04841_b200 import (SU2, Mixer, QaoaParams, QaoaSimulator, TermPolynomial, hamming_weight_state,
                                   labs_terms, maxcut_terms, qaoa_objective, simulate_qaoa, triangle_graph,
                                   uniform_state)
from paper_2309_04841_b200 import instrumentation, mixers, statevec
from paper_2309_04841_b200.costs import DeviceCosts
from paper_2309_04841_b200.problems import portfolio_terms

pytestmark = pytest.mark.gpu

ATOL = 1e-10
SIMS = ["labs8_x_p3", "labs12_x_p4", "labs14_x_p3", "rand5_x_p2", "rand10_x_p5", "cubic12_x_p6",
        "maxcut26sub14_x_p2", "port8_ring_p2", "port8_complete_p2", "port12_ring_p2", "port12_complete_p1",
        "labs8_custom_p2"]


@pytest.mark.parametrize("case", SIMS)
def test_matches_reference_golden(golden, case):
    name = case.split("_")[0]
    n, pairs = golden_terms(golden, name)
    kind = {"x": "x", "ring": "xy-ring", "complete": "xy-complete", "custom": "custom"}[case.split("_")[1]]
    mixer = Mixer.custom(lambda b: [SU2(np.cos(b), np.sin(b))] * n) if kind == "custom" else Mixer(kind)
    initial = hamming_weight_state(n, {8: 4, 12: 6}[n]) if kind.startswith("xy") else None
    sim = QaoaSimulator(terms=TermPolynomial.from_pairs(n, pairs), mixer=mixer)
    res = sim.simulate_qaoa(golden[f"sim/{case}/gammas"], golden[f"sim/{case}/betas"], initial=initial)
    np.testing.assert_allclose(sim.get_statevector(res), golden[f"sim/{case}/state"], rtol=0, atol=ATOL)
    e_ref = float(golden[f"sim/{case}/E"])
    assert sim.get_expectation(res) == pytest.approx(e_ref, rel=1e-10, abs=1e-10)
    assert sim.get_overlap(res) == pytest.approx(float(golden[f"sim/{case}/overlap"]), abs=1e-10)


@pytest.fixture(params=[-1, 0, 1], ids=["plan-auto", "plan-legacy", "plan-smallfuse"])
def pass_plan(request):
    """Run a test under each group plan of the tiled pass program."""
    from paper_2309_04841_b200 import _lib

    _lib.call("fq_set_option", b"plan", request.param)
    yield request.param
    _lib.call("fq_set_option", b"plan", -1)


@pytest.mark.parametrize("n,p,seed", [(13, 1, 0), (13, 3, 1), (14, 2, 2), (16, 4, 3), (17, 5, 4), (19, 3, 5),
                                      (22, 2, 6), (24, 2, 7), (25, 1, 8)])
def test_tiled_x_labs_vs_oracle(n, p, seed, pass_plan):
    """Fused tiled passes (uint16 phase tables, alternating-order layer fusion)."""
    rng = np.random.default_rng(seed)
    g, b = rng.uniform(-1, 1, p), rng.uniform(-1.6, 1.6, p)
    poly = labs_terms(n)
    sim = QaoaSimulator(terms=poly)
    assert sim.device_costs.u16 is not None
    res = sim.simulate_qaoa(g, b)
    costs = sim.get_cost_diagonal()
    ref = O.simulate(costs, g, b)
    got = sim.get_statevector(res)
    # 1e-10 relative to the largest amplitude (amplitudes are ~2^-n/2)
    np.testing.assert_allclose(got, ref, rtol=0, atol=ATOL * np.abs(ref).max())
    e_ref = O.expectation(ref, costs)
    assert sim.get_expectation(res) == pytest.approx(e_ref, rel=1e-10)
    assert sim.get_expectation(res, costs=costs) == pytest.approx(e_ref, rel=1e-10)


@pytest.mark.parametrize("n,p,seed", [(13, 2, 10), (15, 3, 11), (18, 2, 12)])
def test_tiled_x_float_costs_vs_oracle(n, p, seed, pass_plan):
    """Float-weight diagonal: float64 cost path with sincos in the pass."""
    rng = np.random.default_rng(seed)
    pairs = random_pairs(rng, n, max_terms=3 * n)
    g, b = rng.uniform(-1, 1, p), rng.uniform(-1, 1, p)
    sim = QaoaSimulator(terms=TermPolynomial.from_pairs(n, pairs))
    assert sim.device_costs.u16 is None
    res = sim.simulate_qaoa(g, b)
    costs = sim.get_cost_diagonal()
    ref = O.simulate(costs, g, b)
    np.testing.assert_allclose(sim.get_statevector(res), ref, rtol=0, atol=1e-12)
    assert sim.get_expectation(res) == pytest.approx(O.expectation(ref, costs), rel=1e-10, abs=1e-12)


def test_u16_and_f64_paths_agree():
    n, p = 16, 6
    rng = np.random.default_rng(77)
    g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
    poly = labs_terms(n)
    dc16 = DeviceCosts.from_polynomial(poly)
    dc64 = DeviceCosts(n, f64=dc16.f64)
    a = QaoaSimulator(costs=dc16)
    c = QaoaSimulator(costs=dc64)
    ra, rc = a.simulate_qaoa(g, b), c.simulate_qaoa(g, b)
    np.testing.assert_allclose(ra.state, rc.state, rtol=0, atol=1e-13)
    assert a.get_expectation(ra) == pytest.approx(c.get_expectation(rc), rel=1e-12)


@pytest.mark.parametrize("n", [9, 13, 15])
def test_custom_mixer_random_su2_vs_oracle(n, pass_plan):
    rng = np.random.default_rng(40 + n)
    p = 2
    tables = [[random_su2_coeffs(rng) for _ in range(n)] for _ in range(p)]
    it = iter(range(p))
    fac_calls = {}

    def factory(beta):
        idx = fac_calls.setdefault(beta, len(fac_calls))
        return [SU2(a, b) for a, b in tables[idx]]

    betas = [0.3, 0.9]
    gammas = [0.2, -0.4]
    poly = labs_terms(n)
    sim = QaoaSimulator(terms=poly, mixer=Mixer.custom(factory))
    res = sim.simulate_qaoa(gammas, betas)
    costs = sim.get_cost_diagonal()
    ref = O.simulate(costs, gammas, betas, "custom", None, lambda b: tables[betas.index(b)])
    np.testing.assert_allclose(res.state, ref, rtol=0, atol=1e-12)
    del it


@pytest.mark.parametrize("kind", ["xy-ring", "xy-complete"])
@pytest.mark.parametrize("n", [6, 13, 14, 17, 20])
def test_xy_mixers_vs_oracle(kind, n):
    rng = np.random.default_rng(n)
    p = 2
    g, b = rng.uniform(-1, 1, p), rng.uniform(-1, 1, p)
    poly = portfolio_terms(n)
    init = hamming_weight_state(n, n // 2)
    sim = QaoaSimulator(terms=poly, mixer=kind)
    res = sim.simulate_qaoa(g, b, initial=init)
    costs = sim.get_cost_diagonal()
    ref = O.simulate(costs, g, b, kind, O.hamming_weight_state(n, n // 2))
    np.testing.assert_allclose(res.state, ref, rtol=0, atol=1e-12)
    w = np.bitwise_count(np.arange(1 << n, dtype=np.uint64))
    assert np.sum(np.abs(res.state[w != n // 2]) ** 2) < 1e-20


@pytest.mark.parametrize("kind", ["xy-ring", "xy-complete"])
@pytest.mark.parametrize("n,p", [(13, 1), (16, 2), (19, 1), (22, 1)])
def test_tiled_xy_random_state_and_per_gate_path(kind, n, p):
    """Tiled XY passes (gate-sequence scheduler, register rounds, swizzled
    transposes) on a random complex initial state with float64 costs, against
    the oracle and against the one-kernel-per-gate path (option xy_tiled=0)."""
    from paper_2309_04841_b200 import _lib

    rng = np.random.default_rng(100 + n)
    g, b = rng.uniform(-1, 1, p), rng.uniform(-1.6, 1.6, p)
    init = random_state(rng, n)
    poly = TermPolynomial.from_pairs(n, random_pairs(rng, n, max_terms=2 * n))
    sim = QaoaSimulator(terms=poly, mixer=kind)
    res = sim.simulate_qaoa(g, b, initial=init)
    costs = sim.get_cost_diagonal()
    ref = O.simulate(costs, g, b, kind, np.array(init))
    np.testing.assert_allclose(res.state, ref, rtol=0, atol=1e-12)
    assert sim.get_expectation(res) == pytest.approx(O.expectation(ref, costs), rel=1e-10, abs=1e-12)
    _lib.call("fq_set_option", b"xy_tiled", 0)
    try:
        res0 = sim.simulate_qaoa(g, b, initial=init)
    finally:
        _lib.call("fq_set_option", b"xy_tiled", 1)
    np.testing.assert_allclose(res.state, res0.state, rtol=0, atol=1e-12)


def test_batched_small_n_matches_single():
    poly = labs_terms(12)
    sim = QaoaSimulator(terms=poly)
    rng = np.random.default_rng(5)
    G, B = rng.uniform(0, 1, (40, 4)), rng.uniform(0, 1, (40, 4))
    got = sim.simulate_qaoa_batched(G, B)
    costs = sim.get_cost_diagonal()
    for i in range(0, 40, 7):
        ref = O.expectation(O.simulate(costs, G[i], B[i]), costs)
        assert got[i] == pytest.approx(ref, rel=1e-11)


def test_long_program_chunks_and_norm():
    # > 512 layers forces chunked resident launches; norm preserved (ref test_qaoa.py:92-97)
    rng = np.random.default_rng(13)
    poly = labs_terms(10)
    p = 600
    res = simulate_qaoa(poly, QaoaParams(tuple(rng.uniform(-1, 1, p)), tuple(rng.uniform(-1, 1, p))))
    assert np.linalg.norm(res.state) == pytest.approx(1.0, abs=1e-10)
    poly = labs_terms(14)
    p = 40
    res = simulate_qaoa(poly, QaoaParams(tuple(rng.uniform(-1, 1, p)), tuple(rng.uniform(-1, 1, p))))
    assert np.linalg.norm(res.state) == pytest.approx(1.0, abs=1e-10)


def test_gamma_zero_layers_and_beta_special_values():
    # gamma == 0 must skip the phase, beta near pi/2 exercises the (cot, 1) form
    n = 15
    poly = labs_terms(n)
    sim = QaoaSimulator(terms=poly)
    g = [0.0, 0.3, 0.0, 0.2]
    b = [np.pi / 2, 0.3, 1.2, -2.0]
    res = sim.simulate_qaoa(g, b)
    costs = sim.get_cost_diagonal()
    ref = O.simulate(costs, g, b)
    np.testing.assert_allclose(res.state, ref, rtol=0, atol=1e-12)


# ------------------------------------------------------------------ reference API contract
def test_zero_layers_and_objective():
    poly = maxcut_terms(triangle_graph())
    res = simulate_qaoa(poly, QaoaParams((), ()))
    np.testing.assert_array_equal(res.state, uniform_state(3))
    assert qaoa_objective(poly, QaoaParams((), ())) == pytest.approx(-1.5)
    assert qaoa_objective(poly, QaoaParams((0.0,), (0.7,))) == pytest.approx(-1.5, abs=1e-12)


def test_accessors_and_overrides():
    poly = maxcut_terms(triangle_graph())
    sim = QaoaSimulator(terms=poly)
    res = sim.simulate_qaoa((), ())
    np.testing.assert_array_equal(sim.get_statevector(res), uniform_state(3))
    np.testing.assert_allclose(sim.get_probabilities(res), np.full(8, 1 / 8))
    assert sim.get_expectation(res) == pytest.approx(-1.5)
    assert sim.get_overlap(res) == pytest.approx(6 / 8)
    np.testing.assert_array_equal(sim.get_cost_diagonal(), [0, -2, -2, -2, -2, -2, -2, 0])
    other = np.arange(8, dtype=float)
    assert sim.get_expectation(res, costs=other) == pytest.approx(3.5)
    assert sim.get_overlap(res, costs=other) == pytest.approx(1 / 8)


def test_precompute_once_and_memo():
    poly = TermPolynomial.from_pairs(6, [(1.25, (0, 3)), (0.75, (1, 4, 5))])
    instrumentation.reset()
    sim = QaoaSimulator(terms=poly)
    assert instrumentation.get("precompute") == 1
    sim.simulate_qaoa((0.1,), (0.2,))
    sim.simulate_qaoa((0.3,), (0.4,))
    assert instrumentation.get("precompute") == 1
    poly2 = TermPolynomial.from_pairs(5, [(1.0625, (0, 2)), (-0.375, (1, 3, 4))])
    instrumentation.reset()
    for a in (0.1, 0.5, 0.7):
        qaoa_objective(poly2, QaoaParams((a,), (a + 0.1,)))
    assert instrumentation.get("precompute") == 1


def test_errors_match_reference():
    with pytest.raises(ValueError, match="exactly one"):
        QaoaSimulator(terms=TermPolynomial(2), costs=np.zeros(4))
    with pytest.raises(ValueError, match="exactly one"):
        QaoaSimulator()
    with pytest.raises(ValueError, match="initial"):
        simulate_qaoa(labs_terms(4), QaoaParams((0.1,), (0.2,)), mixer="xy-ring")
    with pytest.raises(ValueError, match="cost vector"):
        statevec.expectation(uniform_state(3), np.zeros(4))
    with pytest.raises(ValueError, match="out of range"):
        mixers.apply_su2(uniform_state(3), SU2.identity(), 3)
    with pytest.raises(ValueError, match="distinct"):
        mixers.apply_xy(uniform_state(3), 0.1, 1, 1)


def test_statevec_goldens_host_in_place():
    st = uniform_state(2)
    statevec.apply_phase(st, np.ones(4), np.pi)
    np.testing.assert_allclose(st, np.full(4, -0.5), atol=1e-15)
    st = uniform_state(2)
    statevec.apply_phase(st, np.array([1.0, -1.0, -1.0, 1.0]), np.pi / 2)
    np.testing.assert_allclose(st, [-0.5j, 0.5j, 0.5j, -0.5j], atol=1e-15)
    st = uniform_state(3)
    before = st.copy()
    statevec.apply_phase(st, np.arange(8.0), 0.0)
    np.testing.assert_array_equal(st, before)
    probs = statevec.probabilities(st, preserve_state=False)
    assert np.shares_memory(probs, st)
    np.testing.assert_allclose(probs, np.full(8, 1 / 8))


def test_layer_functions_vs_oracle():
    rng = np.random.default_rng(2)
    for n in (5, 14):
        x = random_state(rng, n)
        ref = x.copy()
        O.rx_layer(ref, 0.37)
        got = x.copy()
        mixers.rx_layer(got, 0.37)
        np.testing.assert_allclose(got, ref, atol=1e-13)
        for kind, fn in (("xy-ring", mixers.xy_ring_layer), ("xy-complete", mixers.xy_complete_layer)):
            ref = x.copy()
            O.mixer_layer(ref, kind, 0.41)
            got = x.copy()
            fn(got, 0.41)
            np.testing.assert_allclose(got, ref, atol=1e-13)


def test_device_tensor_inputs():
    n = 14
    psi = uniform_state(n, device=True)
    assert isinstance(psi, torch.Tensor) and psi.is_cuda
    mixers.rx_layer(psi, 0.2)
    ref = O.uniform_state(n)
    O.rx_layer(ref, 0.2)
    np.testing.assert_allclose(psi.cpu().numpy(), ref, atol=1e-13)


def test_custom_mixer_zero_layers():
    """Zero layers under a custom mixer (found by scripts/stress.py): the uniform state."""
    from paper_2309_04841_b200 import SU2, Mixer

    for n in (5, 14):
        sim = QaoaSimulator(terms=labs_terms(n), mixer=Mixer.custom(lambda beta: [SU2.rx(beta)] * n))
        res = sim.simulate_qaoa([], [])
        np.testing.assert_allclose(res.state, np.full(1 << n, 2 ** (-n / 2)), rtol=0, atol=1e-15)


@pytest.mark.parametrize("n,p", [(12, 100), (11, 200)])
def test_custom_mixer_deep_resident_program(n, p):
    """Custom SU(2) layers beyond one scratch chunk on the one-CTA (n <= 12)
    path: p * n * 4 doubles exceed FQ_SCRATCH_DOUBLES, so the program runs in
    several launches (it used to raise).  The reference takes any p."""
    from paper_2309_04841_b200 import SU2, Mixer

    rng = np.random.default_rng(n + p)
    gammas = list(rng.uniform(-0.2, 0.2, p))
    betas = list(rng.uniform(0.0, 1.0, p))

    def factory(beta):
        return [SU2(np.cos(beta + 0.01 * q), -1j * np.sin(beta + 0.01 * q)) for q in range(n)]

    sim = QaoaSimulator(terms=labs_terms(n), mixer=Mixer.custom(factory))
    res = sim.simulate_qaoa(gammas, betas)
    costs = sim.get_cost_diagonal()
    ref = O.simulate(costs, gammas, betas, "custom", None, lambda b: [(u.a, u.b) for u in factory(b)])
    np.testing.assert_allclose(res.state, ref, rtol=0, atol=1e-10)
    assert sim.get_expectation(res) == pytest.approx(O.expectation(ref, costs), rel=1e-10)
