"""The register-round resident kernel (n <= 12, X and custom SU(2) mixers,
csrc/evolve.cu k_resident16) against the CPU oracle (reference qaoa.py:137-149
loop, _kernels.py:14-27 / 68-73) at every n = 1..12, even and odd depths,
uint16 phase tables and float64 sincos phases, explicit initial states,
gamma = 0 layers, and the batched launch (one parameter set per CTA) — and
against the previous one-sweep-per-qubit kernel (option res16 = 0)."""

import numpy as np
import pytest

from _helpers import random_state
from oracle import oracle as O
from paper_2309_04841_b200 import SU2, Mixer, QaoaSimulator, TermPolynomial, _lib, labs_terms

pytestmark = pytest.mark.gpu

ATOL = 1e-10


@pytest.fixture
def res16_off():
    _lib.call("fq_set_option", b"res16", 0)
    yield
    _lib.call("fq_set_option", b"res16", 2)  # the default (k_resident8)


def _float_poly(n, seed):
    rng = np.random.default_rng(seed)
    pairs = [(float(rng.normal()), tuple(int(q) for q in rng.choice(n, size=int(rng.integers(1, min(n, 3) + 1)),
                                                                      replace=False)))
             for _ in range(3 * n)]
    return TermPolynomial.from_pairs(n, pairs)


@pytest.mark.parametrize("n", list(range(1, 13)))
@pytest.mark.parametrize("p", [0, 1, 4, 5])
def test_x_labs_vs_oracle(n, p):
    rng = np.random.default_rng(100 * n + p)
    g, b = rng.uniform(-1, 1, p), rng.uniform(-1.6, 1.6, p)
    sim = QaoaSimulator(terms=labs_terms(n)) if n >= 2 else QaoaSimulator(terms=_float_poly(1, 1))
    res = sim.simulate_qaoa(g, b)
    costs = sim.get_cost_diagonal()
    ref = O.simulate(costs, g, b)
    np.testing.assert_allclose(res.state, ref, rtol=0, atol=ATOL)
    assert sim.get_expectation(res) == pytest.approx(O.expectation(ref, costs), rel=1e-10, abs=1e-12)


@pytest.mark.parametrize("n,p", [(3, 2), (7, 3), (12, 4), (12, 7)])
def test_float_costs_and_initial_state(n, p):
    rng = np.random.default_rng(n * p)
    g, b = rng.uniform(-1, 1, p), rng.uniform(-1.6, 1.6, p)
    g[1 % p] = 0.0  # a gamma = 0 layer skips its phase
    sim = QaoaSimulator(terms=_float_poly(n, n))
    assert sim.device_costs.u16 is None  # float weights: sincos phase per amplitude
    init = random_state(rng, n)
    res = sim.simulate_qaoa(g, b, initial=init)
    costs = sim.get_cost_diagonal()
    ref = O.simulate(costs, g, b, "x", init)
    np.testing.assert_allclose(res.state, ref, rtol=0, atol=ATOL)


@pytest.mark.parametrize("n,p", [(5, 3), (12, 4), (12, 9)])
def test_custom_mixer_vs_oracle(n, p):
    rng = np.random.default_rng(7 * n + p)
    g, b = rng.uniform(-1, 1, p), rng.uniform(-1, 1, p)

    def factory(beta):
        return [SU2(np.cos(beta + 0.03 * q) * np.exp(0.1j * q), -1j * np.sin(beta + 0.03 * q)) for q in range(n)]

    sim = QaoaSimulator(terms=labs_terms(n), mixer=Mixer.custom(factory))
    res = sim.simulate_qaoa(g, b)
    costs = sim.get_cost_diagonal()
    ref = O.simulate(costs, g, b, "custom", None, lambda bb: [(u.a, u.b) for u in factory(bb)])
    np.testing.assert_allclose(res.state, ref, rtol=0, atol=ATOL)


@pytest.mark.parametrize("n", [4, 9, 12])
def test_same_as_sweep_kernel(n, res16_off):
    """The previous resident kernel (one shared-memory sweep per qubit) agrees."""
    rng = np.random.default_rng(n)
    p = 6
    g, b = rng.uniform(-1, 1, p), rng.uniform(-1.6, 1.6, p)
    sim = QaoaSimulator(terms=labs_terms(n))
    old = sim.simulate_qaoa(g, b).state.copy()
    _lib.call("fq_set_option", b"res16", 1)
    new = sim.simulate_qaoa(g, b).state
    np.testing.assert_allclose(new, old, rtol=0, atol=1e-12)


@pytest.mark.parametrize("n,p", [(6, 3), (12, 4), (12, 1)])
def test_batched_vs_oracle(n, p):
    """One CTA per parameter set, uint16 phase tables (levels passed through
    fq_qaoa_evolve_batched_levels)."""
    rng = np.random.default_rng(n + 31 * p)
    G, B = rng.uniform(-1, 1, (300, p)), rng.uniform(-1.6, 1.6, (300, p))
    sim = QaoaSimulator(terms=labs_terms(n))
    got = sim.simulate_qaoa_batched(G, B)
    costs = sim.get_cost_diagonal()
    for i in range(0, 300, 37):
        ref = O.expectation(O.simulate(costs, G[i], B[i]), costs)
        assert got[i] == pytest.approx(ref, rel=1e-10, abs=1e-12)


@pytest.mark.parametrize("n", [8, 12, 15])
def test_objective_fast_path(n):
    """QaoaSimulator.objective (one fq_qaoa_objective call per evaluation,
    prepared descriptor per depth) equals get_expectation(simulate_qaoa(...))
    and the oracle, across depth changes; mismatched angle lists raise like
    QaoaParams."""
    sim = QaoaSimulator(terms=labs_terms(n))
    costs = sim.get_cost_diagonal()
    rng = np.random.default_rng(n)
    for p in (3, 5, 3, 1):
        g, b = rng.uniform(-1, 1, p), rng.uniform(-1.6, 1.6, p)
        e = sim.objective(g, b)
        assert e == pytest.approx(sim.get_expectation(sim.simulate_qaoa(g, b)), rel=1e-12, abs=1e-13)
        assert e == pytest.approx(O.expectation(O.simulate(costs, g, b), costs), rel=1e-10, abs=1e-12)
    with pytest.raises(ValueError, match="gammas but"):
        sim.objective([0.1, 0.2], [0.3])


@pytest.fixture(params=[2, 1, 0], ids=["resident8", "resident16", "sweep"])
def res_variant(request):
    _lib.call("fq_set_option", b"res16", request.param)
    yield request.param
    _lib.call("fq_set_option", b"res16", 2)


@pytest.mark.parametrize("n", [5, 12])
@pytest.mark.parametrize("float_costs", [False, True])
def test_objective_graph_replay(n, float_costs, res_variant):
    """objective() for n <= 12 replays a captured CUDA graph (fq_objective_graph_*:
    angles H2D from pinned memory, the one-CTA program reading them on the device,
    objective D2H): equal to the eager fq_qaoa_objective path and to the oracle over
    many angle sets (gamma = 0 layers included, both RX forms), a depth change
    (a new graph) and uint16 / float64 diagonals."""
    poly = _float_poly(n, 3) if float_costs else labs_terms(n)
    sim = QaoaSimulator(terms=poly)
    costs = sim.get_cost_diagonal()
    rng = np.random.default_rng(40 + n)
    for p in (4, 4, 4, 7, 4):
        g, b = rng.uniform(-1, 1, p), rng.uniform(-1.6, 1.6, p)
        g[rng.integers(0, p)] = 0.0
        sim.use_graph = True
        e_graph = sim.objective(g, b)
        sim.use_graph = False
        e_eager = sim.objective(g, b)
        assert e_graph == pytest.approx(e_eager, rel=1e-13, abs=1e-14)
        assert e_graph == pytest.approx(O.expectation(O.simulate(costs, g, b), costs), rel=1e-10, abs=1e-12)
    sim.use_graph = True
    assert sim._graph_ctx is not None and sim._graph_ctx[0] == 4
    del sim  # the graph handle is released with the simulator (weakref finalizer)
