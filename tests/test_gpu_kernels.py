"""Operator-layer parity: every libfqaoa kernel vs the CPU oracle (which is
pinned to the reference by test_oracle_golden.py).  Integer/byte/index work
is bit-exact; floating point within 1e-12 (fp64)."""

import numpy as np
import pytest
import torch

from _helpers import golden_terms, random_pairs, random_state, random_su2_coeffs
from oracle import oracle as O
from paper_2309_04841_b200 import _lib
from paper_2309_04841_b200.costs import DeviceCosts
from paper_2309_04841_b200.terms import TermPolynomial, precompute_device

pytestmark = pytest.mark.gpu


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def st():
    return _lib.stream()


@pytest.mark.parametrize("n", [1, 2, 5, 11, 14])
def test_su2_on_pairs_every_qubit(n):
    rng = np.random.default_rng(n)
    for q in range(n):
        a, b = random_su2_coeffs(rng)
        x = random_state(rng, n)
        ref = x.copy()
        O.su2_on_pairs(ref, a, b, q)
        d = dev(x)
        _lib.call("fq_su2_on_pairs", d.data_ptr(), d.numel(), a.real, a.imag, b.real, b.imag, q, st())
        np.testing.assert_allclose(d.cpu().numpy(), ref, rtol=0, atol=1e-14)


@pytest.mark.parametrize("n", [2, 5, 13])
def test_xy_and_swap_every_pair(n):
    rng = np.random.default_rng(10 + n)
    beta = 0.71
    for lo in range(n):
        for hi in range(lo + 1, n):
            x = random_state(rng, n)
            ref = x.copy()
            O.xy_on_pairs(ref, np.cos(beta), np.sin(beta), lo, hi)
            d = dev(x)
            _lib.call("fq_xy_on_pairs", d.data_ptr(), d.numel(), np.cos(beta), np.sin(beta), lo, hi, st())
            np.testing.assert_allclose(d.cpu().numpy(), ref, rtol=0, atol=1e-14)
            ref2 = x.copy()
            O.swap_bits(ref2, lo, hi)
            d = dev(x)
            _lib.call("fq_swap_bits", d.data_ptr(), d.numel(), lo, hi, st())
            np.testing.assert_array_equal(d.cpu().numpy(), ref2)


def test_phase_and_abs2():
    rng = np.random.default_rng(3)
    n = 14
    x = random_state(rng, n)
    c = rng.uniform(-300, 300, 1 << n)
    ref = x.copy()
    O.phase_multiply(ref, c, 0.731)
    d = dev(x)
    _lib.call("fq_phase_multiply", d.data_ptr(), dev(c).data_ptr(), d.numel(), 0.731, st())
    np.testing.assert_allclose(d.cpu().numpy(), ref, rtol=0, atol=1e-13)
    ref = x.copy()
    O.abs2_inplace(ref)
    d = dev(x)
    _lib.call("fq_abs2_inplace", d.data_ptr(), d.numel(), st())
    np.testing.assert_array_equal(d.cpu().numpy(), ref)


@pytest.mark.parametrize("name", ["labs8", "labs12", "labs14", "tri", "cubic12", "maxcut26sub14", "rand5", "rand8",
                                  "rand10", "port8", "port12"])
def test_precompute_bit_exact_vs_reference(golden, name):
    n, pairs = golden_terms(golden, name)
    got = precompute_device(TermPolynomial.from_pairs(n, pairs)).cpu().numpy()
    np.testing.assert_array_equal(got.view(np.uint64), golden[f"diag/{name}"].view(np.uint64))


@pytest.mark.parametrize("seed", range(8))
def test_precompute_random_float_and_integer(seed):
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(3, 17))
    for integer in (False, True):
        pairs = random_pairs(rng, n, max_terms=60, integer=integer)
        ref = O.precompute_cost_vector(n, pairs)
        got = precompute_device(TermPolynomial.from_pairs(n, pairs)).cpu().numpy()
        np.testing.assert_array_equal(got.view(np.uint64), ref.view(np.uint64))


def test_precompute_shard_offsets_and_wide_indices():
    # a slice at a large global base (index bits above 32 exercise the 64-bit mask path)
    pairs = O.labs_terms(36)
    from paper_2309_04841_b200.problems import labs_terms

    poly = labs_terms(36)
    base = (5 << 33) + 12345
    got = precompute_device(poly, index_base=base, size=4096).cpu().numpy()
    ref = O.precompute_cost_vector(36, pairs, base=base, size=4096)
    np.testing.assert_array_equal(got, ref)
    # uint16 levels straight from the terms decode to the same values
    dc = DeviceCosts.from_polynomial(poly, keep_f64=False, index_base=base, n_local=12)
    lv = dc.u16.cpu().numpy().astype(np.float64)
    np.testing.assert_array_equal(dc.scale * lv + dc.offset, ref)


def test_compact_u16_round_trip(golden):
    for name in ("labs14", "cubic12", "maxcut26sub14"):
        dc = DeviceCosts.from_array(golden[f"diag/{name}"])
        assert dc.u16 is not None, name
        dec = dc.scale * dc.u16.cpu().numpy().astype(np.float64) + dc.offset
        np.testing.assert_array_equal(dec, golden[f"diag/{name}"])
    dc = DeviceCosts.from_array(golden["diag/port12"])
    assert dc.u16 is None  # float weights: not on a 16-bit grid


def test_init_states():
    from math import comb, sqrt

    n = 13
    d = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
    _lib.call("fq_init_state", d.data_ptr(), d.numel(), -1, 1 / sqrt(1 << n), 0, st())
    np.testing.assert_array_equal(d.cpu().numpy(), O.uniform_state(n))
    _lib.call("fq_init_state", d.data_ptr(), d.numel(), 6, 1 / sqrt(comb(n, 6)), 0, st())
    np.testing.assert_array_equal(d.cpu().numpy(), O.hamming_weight_state(n, 6))


def test_reductions_vs_oracle():
    rng = np.random.default_rng(9)
    n = 17
    x = random_state(rng, n)
    c = np.rint(rng.uniform(-50, 50, 1 << n))
    dc = DeviceCosts.from_array(c)
    assert dc.u16 is not None
    from paper_2309_04841_b200.statevec import expectation_device, overlap_device

    e_ref = O.expectation(x, c)
    d = dev(x)
    assert float(expectation_device(d, dc).item()) == pytest.approx(e_ref, rel=1e-12, abs=1e-12)
    f = DeviceCosts(n, f64=dev(c))
    assert float(expectation_device(d, f).item()) == pytest.approx(e_ref, rel=1e-12, abs=1e-12)
    assert dc.minmax() == (c.min(), c.max())
    assert float(overlap_device(d, dc, c.min()).item()) == pytest.approx(O.overlap(x, c), abs=1e-14)
    # deterministic: same bits twice
    a = expectation_device(d, dc).item()
    b = expectation_device(d, dc).item()
    assert a == b


@pytest.mark.parametrize("case", ["labs", "maxcut_halves", "random_int", "dup_masks"])
@pytest.mark.parametrize("n", [12, 15, 20, 25])
def test_wht_diagonal_bit_exact(case, n):
    """Integer / dyadic diagonals as a Walsh-Hadamard transform of the weights
    (fq_precompute_wht) equal the reference's per-element sum bit for bit."""
    import torch

    from paper_2309_04841_b200 import _lib
    from paper_2309_04841_b200.problems import Graph, labs_terms, maxcut_terms
    from paper_2309_04841_b200.terms import term_arrays

    rng = np.random.default_rng(n * 7 + len(case))
    if case == "labs":
        poly = labs_terms(n)
    elif case == "maxcut_halves":
        edges = {tuple(sorted(rng.choice(n, 2, replace=False).tolist())) for _ in range(3 * n)}
        poly = maxcut_terms(Graph.from_edges(n, sorted(edges)))
    elif case == "random_int":
        poly = TermPolynomial.from_pairs(n, random_pairs(rng, n, max_terms=4 * n, integer=True))
    else:  # repeated supports and a constant: the scatter must add them exactly
        pairs = [(float(rng.integers(-9, 10)), (1, 3)) for _ in range(5)] + [(2.5, ()), (-0.25, (0, n - 1))] * 3
        poly = TermPolynomial.from_pairs(n, pairs)
    pairs = [(t.weight, t.support) for t in poly.terms]
    ref = O.precompute_cost_vector(n, pairs)
    ta = term_arrays(poly)
    assert ta.iweights is not None
    out = torch.empty(1 << n, dtype=torch.float64, device="cuda")
    iw, m = torch.from_numpy(ta.iweights).cuda(), torch.from_numpy(ta.masks).cuda()  # alive until the sync below
    _lib.call("fq_precompute_wht", out.data_ptr(), 1 << n, iw.data_ptr(), m.data_ptr(), len(poly.terms), ta.shift, 0,
              _lib.stream())
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint64), ref.view(np.uint64))


def test_wht_diagonal_shards():
    """A shard [r 2^nl, (r+1) 2^nl) folds the global bits into the term signs."""
    from paper_2309_04841_b200.problems import labs_terms

    n, nl = 18, 14
    poly = labs_terms(n)
    pairs = [(t.weight, t.support) for t in poly.terms]
    full = O.precompute_cost_vector(n, pairs)
    for r in range(1 << (n - nl)):
        got = precompute_device(poly, index_base=r << nl, size=1 << nl).cpu().numpy()
        np.testing.assert_array_equal(got.view(np.uint64), full[r << nl:(r + 1) << nl].view(np.uint64))


def test_u16_levels_via_wht_chunks():
    """The uint16-only diagonal (capacity path: no float64 vector) built from
    per-chunk Walsh-Hadamard transforms decodes to the reference diagonal."""
    from paper_2309_04841_b200.problems import labs_terms

    n = 20
    poly = labs_terms(n)
    ref = O.precompute_cost_vector(n, [(t.weight, t.support) for t in poly.terms])
    dc = DeviceCosts.from_polynomial(poly, keep_f64=False)
    assert dc.f64 is None
    lv = dc.u16.cpu().numpy().astype(np.float64)
    np.testing.assert_array_equal(dc.scale * lv + dc.offset, ref)
    # a shard of a larger problem (global bits folded into the term signs)
    dc2 = DeviceCosts.from_polynomial(labs_terms(22), keep_f64=False, index_base=3 << 20, n_local=20)
    ref2 = O.precompute_cost_vector(22, [(t.weight, t.support) for t in labs_terms(22).terms], base=3 << 20, size=1 << 20)
    np.testing.assert_array_equal(dc2.scale * dc2.u16.cpu().numpy().astype(np.float64) + dc2.offset, ref2)
    # levels start at the observed minimum (phase tables sized by the range in use)
    for d, r in ((dc, ref), (dc2, ref2)):
        assert int(d.u16.cpu().numpy().min()) == 0 and d.offset == r.min()
        assert d.levels == int(round((r.max() - r.min()) / d.scale)) + 1


def test_rebase_u16():
    from paper_2309_04841_b200 import _lib

    rng = np.random.default_rng(5)
    for size in (8, 4096 + 5, 1 << 16):
        lv = rng.integers(300, 65335, size).astype(np.uint16)
        t = torch.from_numpy(lv.view(np.int16)).cuda().view(torch.uint16)
        _lib.call("fq_rebase_u16", t.data_ptr(), size, 300, _lib.stream())
        np.testing.assert_array_equal(t.view(torch.int16).cpu().numpy().view(np.uint16), lv - 300)
        # negative delta: levels move up (the sharded common origin)
        _lib.call("fq_rebase_u16", t.data_ptr(), size, -200, _lib.stream())
        np.testing.assert_array_equal(t.view(torch.int16).cpu().numpy().view(np.uint16), lv - 100)
