"""The operator layer under the reference's names (paper_2309_04841_b200._kernels,
mirror of fastqaoa/_kernels.py): every operator on host arrays (in place, as
the numba kernels) and on CUDA tensors, against the oracle's restatement of
the same kernel — bit-exact where the reference's operation order is kept
(swap, abs2, accumulate), 1e-15 otherwise."""

import numpy as np
import pytest
import torch

from _helpers import random_pairs, random_state, random_su2_coeffs
from oracle import oracle as O
from paper_2309_04841_b200 import _kernels as K

pytestmark = pytest.mark.gpu


def test_warm_up():
    K.warm_up()


@pytest.mark.parametrize("n", [2, 5, 13])
def test_operators_host_and_device_vs_oracle(n):
    rng = np.random.default_rng(n)
    psi = random_state(rng, n)
    costs = rng.uniform(-3, 3, 1 << n)
    a, b = random_su2_coeffs(rng)
    steps = [
        ("su2_on_pairs", (a, b, n - 1)),
        ("xy_on_pairs", (np.cos(0.3), np.sin(0.3), 0, n - 1)),
        ("swap_bits", (0, n - 1)),
        ("phase_multiply", (costs, 0.7)),
        ("abs2_inplace", ()),
    ]
    host = psi.copy()
    dev = torch.from_numpy(psi.copy()).cuda()
    ref = psi.copy()
    for name, args in steps:
        getattr(K, name)(host, *args)
        dargs = tuple(torch.from_numpy(x).cuda() if isinstance(x, np.ndarray) else x for x in args)
        getattr(K, name)(dev, *dargs)
        getattr(O, name)(ref, *args)
        np.testing.assert_allclose(host, ref, rtol=0, atol=1e-15, err_msg=name)
        np.testing.assert_allclose(dev.cpu().numpy(), ref, rtol=0, atol=1e-15, err_msg=name)


def test_accumulate_terms_bit_exact():
    rng = np.random.default_rng(5)
    n = 11
    pairs = random_pairs(rng, n, max_terms=40)
    w = np.array([p[0] for p in pairs])
    m = np.array([sum(1 << q for q in p[1]) for p in pairs], dtype=np.int64)
    out = rng.uniform(-1, 1, 1 << n)
    ref = out.copy()
    K.accumulate_terms(out, w, m)
    O.accumulate_terms(ref, w, m)
    np.testing.assert_array_equal(out, ref)
    d = torch.zeros(1 << n, dtype=torch.float64, device="cuda")
    K.accumulate_terms(d, w, m)
    np.testing.assert_array_equal(d.cpu().numpy(), O.precompute_cost_vector(n, pairs))


def test_operator_argument_errors():
    psi = np.full(8, 8 ** -0.5, dtype=np.complex128)
    with pytest.raises(ValueError):
        K.phase_multiply(psi, np.zeros(4), 0.1)
    with pytest.raises(ValueError):
        K.su2_on_pairs(psi.astype(np.complex64), 1.0, 0.0, 0)
    with pytest.raises(ValueError):
        K.accumulate_terms(np.zeros(8), np.ones(2), np.ones(3, dtype=np.int64))
