"""Every pass-plan shape the X-mixer planner can choose, pinned.

The planner (csrc/evolve.cu plan_x_search) picks per n among group styles x
high-group chunk sizes tmax = 4..12; above n = 30 (where the reference refuses
to run, terms.py:23,109-113) it takes 4-group plans with 64-256-B runs, and the
sharded program (config 5, LABS n = 34 on 2/4/8 GPUs) runs those shapes with
n_local = 31..33.  Parity for them rests on:

* every forced shape (fq_set_option "plan" x "plan_tmax") against the CPU
  oracle at n = 18..24 (same kernels, same round programs, same run lengths);
* the single-state program against the sharded program (K = 2/4/8 shards) at
  n = 31 complex128 and n = 33 complex64, and K-invariance at n_local = 30
  (reference Alg. 4 / distributed.py:137-153: sharding must not change the
  result).
"""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2309_04841_b200 import QaoaParams, QaoaSimulator, _lib, labs_terms
from paper_2309_04841_b200.problems import portfolio_terms

pytestmark = pytest.mark.gpu

ATOL = 1e-10


@pytest.fixture
def reset_plan():
    yield
    _lib.call("fq_set_option", b"plan", -1)
    _lib.call("fq_set_option", b"plan_tmax", 0)


def _shapes(n, p):
    """Distinct plans over (style, tmax): {description: (style, tmax)}."""
    out = {}
    for style in (0, 1):
        for tmax in range(4, 13):
            _lib.call("fq_set_option", b"plan", style)
            _lib.call("fq_set_option", b"plan_tmax", tmax)
            out.setdefault(_lib.describe_x_plan(n, p), (style, tmax))
    _lib.call("fq_set_option", b"plan", -1)
    _lib.call("fq_set_option", b"plan_tmax", 0)
    return out


@pytest.mark.parametrize("n", [18, 20, 22, 24])
def test_every_plan_shape_vs_oracle_labs(n, reset_plan):
    """uint16 costs (phase tables, cp.async cost slices in the fused passes)."""
    p = 3
    rng = np.random.default_rng(n)
    g, b = rng.uniform(-1, 1, p), rng.uniform(-1.6, 1.6, p)
    sim = QaoaSimulator(terms=labs_terms(n))
    costs = sim.get_cost_diagonal()
    ref = O.simulate(costs, g, b)
    e_ref = O.expectation(ref, costs)
    shapes = _shapes(n, p)
    assert len(shapes) >= 3, shapes
    for desc, (style, tmax) in shapes.items():
        _lib.call("fq_set_option", b"plan", style)
        _lib.call("fq_set_option", b"plan_tmax", tmax)
        res = sim.simulate_qaoa(g, b)
        np.testing.assert_allclose(res.state, ref, rtol=0, atol=ATOL * np.abs(ref).max(), err_msg=desc)
        assert sim.get_expectation(res) == pytest.approx(e_ref, rel=1e-10), desc


@pytest.mark.parametrize("n", [20])
def test_every_plan_shape_vs_oracle_float_costs(n, reset_plan):
    """float64 costs (sincos phase in the pass)."""
    p = 2
    rng = np.random.default_rng(100 + n)
    g, b = rng.uniform(-1, 1, p), rng.uniform(-1, 1, p)
    sim = QaoaSimulator(terms=portfolio_terms(n))
    assert sim.device_costs.u16 is None
    costs = sim.get_cost_diagonal()
    ref = O.simulate(costs, g, b)
    for desc, (style, tmax) in _shapes(n, p).items():
        _lib.call("fq_set_option", b"plan", style)
        _lib.call("fq_set_option", b"plan_tmax", tmax)
        res = sim.simulate_qaoa(g, b)
        np.testing.assert_allclose(res.state, ref, rtol=0, atol=ATOL * np.abs(ref).max(), err_msg=desc)


@pytest.mark.parametrize("n", [20, 22])
def test_every_plan_shape_complex64(n, reset_plan):
    p = 3
    rng = np.random.default_rng(200 + n)
    g, b = np.linspace(0.01, 0.1, p), np.linspace(0.6, 0.06, p)
    sim = QaoaSimulator(terms=labs_terms(n), dtype="complex64")
    costs = sim.get_cost_diagonal()
    ref = O.simulate(costs, g, b)
    e_ref = O.expectation(ref, costs)
    for desc, (style, tmax) in _shapes(n, p).items():
        _lib.call("fq_set_option", b"plan", style)
        _lib.call("fq_set_option", b"plan_tmax", tmax)
        res = sim.simulate_qaoa(g, b)
        np.testing.assert_allclose(res.state, ref, rtol=0, atol=1e-4 * np.abs(ref).max(), err_msg=desc)
        assert sim.get_expectation(res) == pytest.approx(e_ref, rel=1e-4), desc
    del rng


def _sample(n, n_samples=4096, seed=5):
    return np.sort(np.random.default_rng(seed).choice(1 << n, n_samples, replace=False))


def _fingerprint(shards, idx, n_blocks=1024):
    """(|psi|^2 sums over n_blocks contiguous blocks, amplitudes at idx) of a
    state held as one tensor or as K equal shards in index order."""
    import torch

    K = len(shards)
    per = n_blocks // K
    size = shards[0].numel()
    blk = size // per
    # block by block: no full-size temporaries next to a 32-64 GiB state
    blocks = torch.stack([torch.view_as_real(s[r * blk:(r + 1) * blk]).double().pow(2).sum()
                          for s in shards for r in range(per)]).cpu().numpy()
    amp = np.empty(idx.size, dtype=np.complex128)
    for r, s in enumerate(shards):
        sel = (idx // size) == r
        if sel.any():
            loc = torch.from_numpy(idx[sel] % size).to(s.device)
            amp[sel] = s[loc].cpu().numpy()
    return blocks, amp


@pytest.mark.parametrize("n,dtype,Ks,p", [(31, "complex128", (2, 4, 8), 4), (33, "complex64", (8, 2), 3)])
def test_large_n_sharded_equals_single_state(n, dtype, Ks, p):
    """n > 30 (beyond the reference): the single-state program (4-group plan)
    equals the sharded program at every K (n_local = n - log2 K, including
    n_local = 30): block norms and sampled amplitudes to 1e-10 (complex64:
    1e-5 of the largest), objectives to 1e-10 relative (complex64: 1e-5)."""
    import gc

    import torch

    from paper_2309_04841_b200.distributed import simulate_qaoa_distributed

    free, _ = torch.cuda.mem_get_info()
    per_amp = (16 if dtype == "complex128" else 8) + 2
    if free < (1 << n) * per_amp * 1.15:
        pytest.skip(f"needs {(1 << n) * per_amp / 2**30:.0f} GiB of device memory")
    tol = 1e-10 if dtype == "complex128" else 1e-5
    g, b = np.linspace(0.02, 0.08, p), np.linspace(0.5, 0.1, p)
    sim = QaoaSimulator(terms=labs_terms(n), dtype=dtype)
    idx = _sample(n)
    res = sim.simulate_qaoa(g, b)
    e1 = sim.get_expectation(res)
    blocks1, amp1 = _fingerprint([res.state_device], idx)
    assert abs(blocks1.sum() - 1.0) < 1e-6
    del res
    gc.collect()
    torch.cuda.empty_cache()
    for K in Ks:
        dres = simulate_qaoa_distributed(sim.device_costs, QaoaParams(tuple(g), tuple(b)), K, dtype=dtype)
        assert dres.expectation() == pytest.approx(e1, rel=tol), K
        blocks, amp = _fingerprint(dres.sharded.shards, idx)
        np.testing.assert_allclose(blocks, blocks1, rtol=0, atol=tol * blocks1.max(), err_msg=f"K={K}")
        np.testing.assert_allclose(amp, amp1, rtol=0, atol=tol * np.abs(amp1).max(), err_msg=f"K={K}")
        del dres
        gc.collect()
        torch.cuda.empty_cache()


def _last_pass_kinds():
    """(round program, targets) of every pass of the last X program (fq_last_passes)."""
    import ctypes

    info = (ctypes.c_int * (5 * 64))()
    cnt = _lib.load().fq_last_passes(info, None, 64)
    return [(info[5 * i], info[5 * i + 2]) for i in range(cnt)]


@pytest.fixture
def reset_lane():
    yield
    _lib.call("fq_set_option", b"lane3", 1)
    _lib.call("fq_set_option", b"plan", -1)
    _lib.call("fq_set_option", b"plan_tmax", 0)


@pytest.mark.parametrize("dtype", ["complex128", "complex64"])
@pytest.mark.parametrize("style", [0, 1])
def test_lane_butterfly_programs_vs_oracle(dtype, style, reset_lane):
    """9-target high groups (3 low spectators, tile bit 3 a target: the n = 30
    config-3 shape) run the two-pattern round programs with tile bit 3 as warp-
    shuffle butterflies (K_LANE3), light and fused; both RX forms (|tan b| <= 1 and
    > 1), a gamma = 0 layer (two layers in one light pass) -- against the oracle, and
    against the same plan with lane3 off (the 8|0|4 programs)."""
    n, p = 21, 4
    rng = np.random.default_rng(7 + style)
    g = rng.uniform(-1, 1, p)
    g[2] = 0.0
    b = np.array([0.3, 1.3, -0.4, 1.45])
    sim = QaoaSimulator(terms=labs_terms(n), dtype=dtype)
    costs = sim.get_cost_diagonal()
    ref = O.simulate(costs, g, b)
    e_ref = O.expectation(ref, costs)
    tol = ATOL if dtype == "complex128" else 1e-4
    _lib.call("fq_set_option", b"plan", style)
    _lib.call("fq_set_option", b"plan_tmax", 9)
    states = {}
    for lane in (1, 0):
        _lib.call("fq_set_option", b"lane3", lane)
        res = sim.simulate_qaoa(g, b)
        kinds = _last_pass_kinds()
        nine = [sq for sq, t in kinds if t == 9]
        assert nine, kinds
        # SEQ_84 = 1, SEQ_848 = 3 (two patterns) with lane butterflies; 8|0|4 programs without
        assert all((sq in (1, 3)) == bool(lane) for sq in nine), (lane, kinds)
        np.testing.assert_allclose(res.state, ref, rtol=0, atol=tol * np.abs(ref).max(), err_msg=f"lane3={lane}")
        assert sim.get_expectation(res) == pytest.approx(e_ref, rel=tol)
        states[lane] = res.state
    np.testing.assert_allclose(states[1], states[0], rtol=0, atol=(1e-12 if dtype == "complex128" else 1e-5))
