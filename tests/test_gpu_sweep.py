"""L2-resident slab sweeps (csrc/sweep.cuh): two consecutive passes of the
fused program in one HBM round trip.  A sweep must reproduce the two passes
exactly as they run separately (same tile bodies, same arithmetic order), so
the sweep program is compared with the unswept program bit for bit, and both
with the CPU oracle (reference qaoa.py:137-149 loop) at 1e-10."""

import ctypes

import numpy as np
import pytest

from oracle import oracle as O
from paper_2309_04841_b200 import QaoaSimulator, _lib, labs_terms

pytestmark = pytest.mark.gpu


@pytest.fixture
def sweep_opts():
    yield
    for name, v in ((b"sweep", 0), (b"sweep_team", 32), (b"sweep_slab_log2", 23)):
        _lib.call("fq_set_option", name, v)


def _records():
    info = (ctypes.c_int * (5 * 256))()
    cnt = _lib.load().fq_last_passes(info, None, 256)
    return [tuple(info[5 * i:5 * i + 5]) for i in range(cnt)]


def _run(sim, g, b, sweep):
    _lib.call("fq_set_option", b"sweep", 1 if sweep else 0)
    res = sim.simulate_qaoa(g, b)
    recs = _records()
    return res.state_device.clone(), sim.get_expectation(res), recs


@pytest.mark.parametrize("n,p,dtype", [(26, 4, "complex128"), (25, 3, "complex128"), (26, 3, "complex64")])
def test_sweep_equals_separate_passes_and_oracle(n, p, dtype, sweep_opts):
    rng = np.random.default_rng(n + p)
    g, b = rng.uniform(-1, 1, p), rng.uniform(-1.6, 1.6, p)
    sim = QaoaSimulator(terms=labs_terms(n), dtype=dtype)
    s0, e0, r0 = _run(sim, g, b, sweep=False)
    s1, e1, r1 = _run(sim, g, b, sweep=True)
    assert not any(r[0] >= 100 for r in r0)
    assert any(r[0] >= 100 for r in r1), r1  # some pass pairs ran as sweeps
    assert len(r1) < len(r0)
    # identical arithmetic in both programs: bit-identical states; the objective's
    # partial sums group the tiles differently (per team CTA), so only to rounding
    assert bool((s0 == s1).all())
    assert e1 == pytest.approx(e0, rel=1e-12)
    if dtype == "complex128" and n <= 26:
        costs = sim.get_cost_diagonal()
        ref = O.simulate(costs, g, b)
        np.testing.assert_allclose(s1.cpu().numpy(), ref, rtol=0, atol=1e-10 * np.abs(ref).max())
        assert e1 == pytest.approx(O.expectation(ref, costs), rel=1e-10)


@pytest.mark.parametrize("team,slab_log2", [(16, 23), (37, 23), (64, 24), (8, 21)])
def test_sweep_team_shapes(team, slab_log2, sweep_opts):
    """Other team sizes / slab budgets (uneven tile shares, more or fewer
    teams than slabs allow) give the same state."""
    n, p = 26, 3
    rng = np.random.default_rng(7)
    g, b = rng.uniform(-1, 1, p), rng.uniform(-1, 1, p)
    sim = QaoaSimulator(terms=labs_terms(n))
    s0, e0, _ = _run(sim, g, b, sweep=False)
    _lib.call("fq_set_option", b"sweep_team", team)
    _lib.call("fq_set_option", b"sweep_slab_log2", slab_log2)
    s1, e1, r1 = _run(sim, g, b, sweep=True)
    _lib.call("fq_set_option", b"sweep", 0)
    swept = any(r[0] >= 100 for r in r1)
    assert swept == (slab_log2 >= 23)  # n = 26 slabs are 8 MiB
    assert bool((s0 == s1).all()) and e1 == pytest.approx(e0, rel=1e-12)
