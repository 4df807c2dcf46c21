"""Operator layer with the reference's names and signatures (mirror of
fastqaoa/_kernels.py:14-118): each function mutates its first argument in
place, as the numba kernels do.

Arguments may be CUDA tensors (operated on in place on the current stream,
no copies) or host numpy arrays (copied to the GPU, transformed by the same
libfqaoa kernel, and written back — the reference's in-place contract).  The
simulator itself does not call these per qubit: ``simulate_qaoa`` runs the
fused program (``fq_qaoa_evolve``); these are the per-operator entry points
for code written against ``fastqaoa._kernels``.  No CPU fallback: without a
CUDA device every function raises.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .statevec import _OnDevice

__all__ = ["su2_on_pairs", "xy_on_pairs", "swap_bits", "phase_multiply", "accumulate_terms", "abs2_inplace",
           "warm_up"]


def su2_on_pairs(psi, a, b, q: int) -> None:
    """Pairs (l0, l0 | 2^q): y0 = a x0 - conj(b) x1, y1 = b x0 + conj(a) x1
    (reference _kernels.py:14-27)."""
    a, b = complex(a), complex(b)
    with _OnDevice(psi) as d:
        _lib.call("fq_su2_on_pairs", d.data_ptr(), d.numel(), a.real, a.imag, b.real, b.imag, int(q), _lib.stream())


def xy_on_pairs(psi, cos_b: float, sin_b: float, p_lo: int, p_hi: int) -> None:
    """exp(-i beta (XX + YY)/2) on qubits p_lo < p_hi (reference _kernels.py:30-48)."""
    with _OnDevice(psi) as d:
        _lib.call("fq_xy_on_pairs", d.data_ptr(), d.numel(), float(cos_b), float(sin_b), int(p_lo), int(p_hi),
                  _lib.stream())


def swap_bits(psi, p_lo: int, p_hi: int) -> None:
    """Exchange the amplitudes of index bits p_lo and p_hi (reference _kernels.py:51-65)."""
    with _OnDevice(psi) as d:
        _lib.call("fq_swap_bits", d.data_ptr(), d.numel(), int(p_lo), int(p_hi), _lib.stream())


def _f64_device(x):
    """(device float64 tensor, host array to write back or None)."""
    if isinstance(x, torch.Tensor):
        if not x.is_cuda or x.dtype != torch.float64 or not x.is_contiguous():
            raise ValueError("device arrays must be contiguous CUDA float64 tensors")
        return x, None
    arr = np.asarray(x)
    if arr.dtype != np.float64:
        raise ValueError("host arrays must be float64")
    return torch.from_numpy(np.ascontiguousarray(arr)).to(_lib.device()), arr


def phase_multiply(psi, costs, gamma: float) -> None:
    """psi[k] *= exp(-i gamma costs[k]) (reference _kernels.py:68-73)."""
    c, _ = _f64_device(costs)
    with _OnDevice(psi) as d:
        if c.numel() != d.numel():
            raise ValueError(f"state has {d.numel()} amplitudes but cost vector has {c.numel()} entries")
        _lib.call("fq_phase_multiply", d.data_ptr(), c.data_ptr(), d.numel(), float(gamma), _lib.stream())


def accumulate_terms(out, weights, masks) -> None:
    """out[k] += sum_t weights[t] (-1)^popcount(k & masks[t]), per element
    left to right in term order (reference _kernels.py:76-94)."""
    o, host = _f64_device(out)
    w = torch.as_tensor(np.ascontiguousarray(weights, dtype=np.float64)).to(o.device)
    m = torch.as_tensor(np.ascontiguousarray(masks, dtype=np.int64)).to(o.device)
    if w.numel() != m.numel():
        raise ValueError(f"{w.numel()} weights but {m.numel()} masks")
    if o.numel():
        _lib.call("fq_accumulate_terms", o.data_ptr(), o.numel(), w.data_ptr(), m.data_ptr(), w.numel(), 0,
                  _lib.stream())
    if host is not None:
        host[...] = o.cpu().numpy().reshape(host.shape)


def abs2_inplace(psi) -> None:
    """psi[k] = |psi[k]|^2 + 0j (reference _kernels.py:97-102)."""
    with _OnDevice(psi) as d:
        _lib.call("fq_abs2_inplace", d.data_ptr(), d.numel(), _lib.stream())


def warm_up() -> None:
    """Load libfqaoa, create the device context and run every operator once
    on tiny inputs (reference _kernels.py:105-118: there, numba JIT).  Call
    before timing anything."""
    psi = torch.full((4,), 0.5, dtype=torch.complex128, device=_lib.device())
    costs = torch.zeros(4, dtype=torch.float64, device=_lib.device())
    su2_on_pairs(psi, 1.0 + 0j, 0j, 0)
    xy_on_pairs(psi, 1.0, 0.0, 0, 1)
    swap_bits(psi, 0, 1)
    phase_multiply(psi, costs, 0.0)
    accumulate_terms(costs, np.zeros(1), np.zeros(1, dtype=np.int64))
    abs2_inplace(psi)
    torch.cuda.synchronize()
