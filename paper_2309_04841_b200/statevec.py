"""State-vector construction, diagonal phase and observables on the GPU.

Mirror of the reference's ``fastqaoa.statevec`` (pkg/src/fastqaoa/statevec.py).
Every operation runs through libfqaoa.  Functions accept either a CUDA
``torch.complex128`` tensor (operated on in place, on the current stream) or a
host ``numpy`` array (copied to the device, operated on, and written back in
place, so the reference's in-place contract holds for host callers too).

Qubit i is bit i of an index (reference statevec.py:3-4).
"""

from __future__ import annotations

from math import comb, sqrt

import numpy as np
import torch
from torch.autograd.graph import increment_version

from . import _lib
from .terms import MAX_DENSE_QUBITS, _infer_n


def num_qubits(state) -> int:
    """reference statevec.py:17-19"""
    size = state.numel() if isinstance(state, torch.Tensor) else np.asarray(state).size
    return _infer_n(size)


def _alloc(n: int) -> torch.Tensor:
    return torch.empty(1 << n, dtype=torch.complex128, device=_lib.device())


def uniform_state_device(n: int) -> torch.Tensor:
    if n < 1:
        raise ValueError(f"qubit count must be positive, got {n}")
    psi = _alloc(n)
    _lib.call("fq_init_state", psi.data_ptr(), psi.numel(), -1, 1.0 / sqrt(1 << n), 0, _lib.stream())
    return psi


def uniform_state(n: int, device: bool = False):
    """Equal superposition (reference statevec.py:22-29).  Host array by
    default (drop-in); ``device=True`` returns the CUDA tensor."""
    if n < 1:
        raise ValueError(f"qubit count must be positive, got {n}")
    if device:
        return uniform_state_device(n)
    if n > MAX_DENSE_QUBITS:
        raise MemoryError(f"state vector for n={n} exceeds the dense-size limit")
    return uniform_state_device(n).cpu().numpy()


def basis_state(n: int, k: int) -> np.ndarray:
    """Computational basis state |k> (reference statevec.py:32-38)."""
    if not 0 <= k < (1 << n):
        raise ValueError(f"index {k} out of range for {n} qubits")
    state = np.zeros(1 << n, dtype=np.complex128)
    state[k] = 1.0
    return state


def hamming_weight_state_device(n: int, weight: int, index_base: int = 0, n_local: int | None = None) -> torch.Tensor:
    n_local = n if n_local is None else n_local
    psi = _alloc(n_local)
    _lib.call("fq_init_state", psi.data_ptr(), psi.numel(), weight, 1.0 / sqrt(comb(n, weight)), index_base,
              _lib.stream())
    return psi


def hamming_weight_state(n: int, weight: int, device: bool = False):
    """Uniform superposition over popcount == weight (reference statevec.py:41-54)."""
    if not 0 <= weight <= n:
        raise ValueError(f"weight {weight} out of range for {n} qubits")
    psi = hamming_weight_state_device(n, weight)
    return psi if device else psi.cpu().numpy()


def norm(state) -> float:
    if isinstance(state, torch.Tensor):
        return float(torch.linalg.vector_norm(state).item())
    return float(np.linalg.norm(state))


# ------------------------------------------------------------------ host <-> device adapter
class _OnDevice:
    """Context: yields a CUDA complex128 view of ``state``; writes back to a
    host array on exit (in-place semantics for numpy callers)."""

    def __init__(self, state, write_back: bool = True):
        self.state = state
        self.write_back = write_back
        self.dev = None

    def __enter__(self) -> torch.Tensor:
        if isinstance(self.state, torch.Tensor):
            if not self.state.is_cuda or self.state.dtype != torch.complex128 or not self.state.is_contiguous():
                raise ValueError("device states must be contiguous CUDA complex128 tensors")
            self.dev = self.state
        else:
            arr = np.asarray(self.state)
            if arr.dtype != np.complex128:
                raise ValueError("host states must be complex128 arrays")
            self.dev = torch.from_numpy(np.ascontiguousarray(arr)).to(_lib.device())
        return self.dev

    def __exit__(self, *exc):
        if exc[0] is None and self.write_back:
            if isinstance(self.state, torch.Tensor):
                # the kernels write through raw pointers: record the in-place
                # update in the tensor's version counter so cached observables
                # of a QaoaResult holding it are invalidated
                increment_version(self.state)
            else:
                np.copyto(self.state, self.dev.cpu().numpy())
        return False


def _costs_f64(costs) -> torch.Tensor:
    if isinstance(costs, torch.Tensor):
        return costs.to(device=_lib.device(), dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(costs, dtype=np.float64)).to(_lib.device())


def _size(x) -> int:
    return x.numel() if isinstance(x, torch.Tensor) else np.asarray(x).size


def _check_match(state, costs) -> None:
    if _size(state) != _size(costs):
        raise ValueError(
            f"state has {_size(state)} amplitudes but cost vector has {_size(costs)} entries"
        )


def apply_phase(state, costs, gamma: float) -> None:
    """psi[k] *= exp(-i gamma costs[k]) in place (reference statevec.py:69-78;
    gamma == 0 is a bit-exact no-op)."""
    _check_match(state, costs)
    if gamma == 0.0:
        return
    with _OnDevice(state) as psi:
        c = _costs_f64(costs)
        _lib.call("fq_phase_multiply", psi.data_ptr(), c.data_ptr(), psi.numel(), float(gamma), _lib.stream())


def probabilities(state, preserve_state: bool = True):
    """|amplitude|^2 (reference statevec.py:81-91).  With preserve_state=False
    the squares overwrite the state and its real view is returned."""
    if isinstance(state, torch.Tensor):
        with _OnDevice(state, write_back=not preserve_state) as psi:
            work = psi if not preserve_state else psi.clone()
            _lib.call("fq_abs2_inplace", work.data_ptr(), work.numel(), _lib.stream())
            return torch.view_as_real(work)[:, 0]
    with _OnDevice(state, write_back=not preserve_state) as psi:
        work = psi if not preserve_state else psi.clone()
        _lib.call("fq_abs2_inplace", work.data_ptr(), work.numel(), _lib.stream())
        if preserve_state:
            return torch.view_as_real(work)[:, 0].cpu().numpy()
    return state.real


def expectation_device(psi: torch.Tensor, dc) -> torch.Tensor:
    """sum_k c_k |psi_k|^2 into a 1-element device tensor (no host sync)."""
    out = torch.empty(1, dtype=torch.float64, device=psi.device)
    kind, cp, scale, offset = dc.kernel_view()
    fn = "fq_expectation_c64" if psi.dtype == torch.complex64 else "fq_expectation"
    _lib.call(fn, psi.data_ptr(), cp, kind, scale, offset, psi.numel(), out.data_ptr(),
              _lib.scratch().data_ptr(), _lib.stream())
    return out


def expectation(state, costs) -> float:
    """<state| diag(costs) |state> (reference statevec.py:94-97)."""
    from .costs import DeviceCosts

    _check_match(state, costs)
    with _OnDevice(state, write_back=False) as psi:
        dc = costs if isinstance(costs, DeviceCosts) else DeviceCosts(num_qubits(psi), f64=_costs_f64(costs))
        return float(expectation_device(psi, dc).item())


def overlap_device(psi: torch.Tensor, dc, cutoff: float) -> torch.Tensor:
    out = torch.empty(1, dtype=torch.float64, device=psi.device)
    kind, cp, scale, offset = dc.kernel_view()
    fn = "fq_masked_probability_c64" if psi.dtype == torch.complex64 else "fq_masked_probability"
    _lib.call(fn, psi.data_ptr(), cp, kind, scale, offset, psi.numel(), float(cutoff),
              out.data_ptr(), _lib.scratch().data_ptr(), _lib.stream())
    return out


def overlap(state, costs, tol: float = 0.0) -> float:
    """Probability on minimum-cost states, ties included, clamped to [0, 1]
    (reference statevec.py:100-111)."""
    from .costs import DeviceCosts

    _check_match(state, costs)
    with _OnDevice(state, write_back=False) as psi:
        dc = costs if isinstance(costs, DeviceCosts) else DeviceCosts(num_qubits(psi), f64=_costs_f64(costs))
        lo, _ = dc.minmax()
        total = float(overlap_device(psi, dc, lo + tol).item())
    return min(max(total, 0.0), 1.0)


def save_state(state, path: str) -> None:
    """Little-endian interleaved complex128 dump (reference statevec.py:114-117)."""
    arr = state.cpu().numpy() if isinstance(state, torch.Tensor) else state
    np.ascontiguousarray(arr, dtype="<c16").tofile(path)


def load_state(path: str) -> np.ndarray:
    state = np.fromfile(path, dtype="<c16").astype(np.complex128)
    _infer_n(state.size)
    return state
