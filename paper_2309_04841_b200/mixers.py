"""Mixing operators on the GPU (mirror of reference fastqaoa/mixers.py).

Gate orders are part of the public contract (reference mixers.py:5-15):

* uniform transforms act on qubits 0..n-1 (they commute; any order is the
  same operator, which is what lets the fused kernels batch 12 per pass);
* the XY ring layer applies (0,1), (2,3), ... then (1,2), (3,4), ... and finally
  the wrap pair (n-1, 0) (omitted for n=2);
* the XY complete layer applies all pairs (i, j), i < j, lexicographically.

Every layer-level function runs through ``fq_qaoa_evolve`` (one fused
program, no phase) so it takes the same batched-pass kernels as the
simulator; ``apply_su2`` / ``apply_xy`` map to the single-gate kernels.
"""

from __future__ import annotations

import ctypes
from cmath import cos, sin
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np
import torch
from torch.autograd.graph import increment_version

from . import _lib
from .statevec import _OnDevice, num_qubits


@dataclass(frozen=True)
class SU2:
    """[[a, -conj(b)], [b, conj(a)]] (reference mixers.py:30-58)."""

    a: complex
    b: complex

    def __post_init__(self) -> None:
        det = abs(self.a) ** 2 + abs(self.b) ** 2
        if abs(det - 1.0) > 1e-12:
            raise ValueError(f"matrix is not special unitary: |a|^2+|b|^2 = {det}")

    @classmethod
    def identity(cls) -> SU2:
        return cls(1.0 + 0j, 0j)

    @classmethod
    def rx(cls, beta: float) -> SU2:
        """exp(-i beta X) = cos(beta) I - i sin(beta) X."""
        return cls(cos(beta), -1j * sin(beta))

    def dagger(self) -> SU2:
        return SU2(self.a.conjugate(), -self.b)

    def matrix(self) -> np.ndarray:
        return np.array([[self.a, -self.b.conjugate()], [self.b, self.a.conjugate()]], dtype=np.complex128)


def ring_edges(n: int) -> list[tuple[int, int]]:
    """reference mixers.py:109-118"""
    if n < 2:
        raise ValueError(f"ring mixer needs at least 2 qubits, got {n}")
    if n == 2:
        return [(0, 1)]
    edges = [(q, q + 1) for q in range(0, n - 1, 2)]
    edges += [(q, q + 1) for q in range(1, n - 1, 2)]
    edges.append((n - 1, 0))
    return edges


def complete_edges(n: int) -> list[tuple[int, int]]:
    """reference mixers.py:121-125"""
    if n < 2:
        raise ValueError(f"complete mixer needs at least 2 qubits, got {n}")
    return [(i, j) for i in range(n) for j in range(i + 1, n)]


def su2_table(layers_us: Sequence[Sequence[SU2]]) -> np.ndarray:
    """[layers][n][4] = (a.re, a.im, b.re, b.im) for the custom-mixer kernels."""
    if len(layers_us) == 0:
        return np.zeros((0, 0, 4), dtype=np.float64)
    return np.array([[(complex(u.a).real, complex(u.a).imag, complex(u.b).real, complex(u.b).imag) for u in us]
                     for us in layers_us], dtype=np.float64).reshape(len(layers_us), -1, 4)


def run_program(psi, n: int, mixer: str, layers: Sequence[tuple], dc=None, su2: np.ndarray | None = None,
                init: bool = False, init_amp: float = 0.0, expectation_out=None) -> None:
    """Enqueue one fused program on the current stream.

    ``layers`` = [(gamma, beta, apply_phase, q_lo, q_hi)].  ``dc`` is a
    DeviceCosts (needed when a phase or the expectation is requested)."""
    arr = (_lib.FqLayer * max(1, len(layers)))()
    for i, (g, b, ph, lo, hi) in enumerate(layers):
        arr[i] = _lib.FqLayer(float(g), float(b), int(ph), int(lo), int(hi))
    desc = _lib.FqEvolveDesc()
    desc.psi = psi.data_ptr()
    desc.n = n
    if dc is not None:
        kind, cp, scale, offset = dc.kernel_view()
        desc.cost_kind, desc.costs, desc.cost_scale, desc.cost_offset = kind, cp, scale, offset
        desc.cost_levels = dc.levels if kind == _lib.COST_U16 else 0
    desc.mixer = _lib.MIXER_CODES[mixer]
    desc.n_layers = len(layers)
    desc.layers = arr
    su2_keep = None
    if su2 is not None:
        su2_keep = np.ascontiguousarray(su2, dtype=np.float64)
        desc.su2 = su2_keep.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    desc.init = 1 if init else 0
    desc.init_amp = init_amp
    desc.expectation_dev = expectation_out.data_ptr() if expectation_out is not None else None
    desc.scratch = _lib.scratch().data_ptr()
    desc.state_kind = _lib.STATE_C64 if psi.dtype == torch.complex64 else _lib.STATE_C128
    _lib.check(_lib.load().fq_qaoa_evolve(ctypes.byref(desc), _lib.stream()), "fq_qaoa_evolve")
    increment_version(psi)  # written in place through its pointer (see statevec._OnDevice)


def apply_su2(state, u: SU2, q: int) -> None:
    """Rotate qubit q by u in place (reference mixers.py:61-71)."""
    n = num_qubits(state)
    if not 0 <= q < n:
        raise ValueError(f"qubit {q} out of range for {n} qubits")
    a, b = complex(u.a), complex(u.b)
    with _OnDevice(state) as psi:
        _lib.call("fq_su2_on_pairs", psi.data_ptr(), psi.numel(), a.real, a.imag, b.real, b.imag, q, _lib.stream())


def apply_uniform_su2(state, us: Sequence[SU2]) -> None:
    """u[n-1] x ... x u[0] in place (reference mixers.py:74-84)."""
    n = num_qubits(state)
    if len(us) != n:
        raise ValueError(f"expected {n} matrices, got {len(us)}")
    with _OnDevice(state) as psi:
        run_program(psi, n, "custom", [(0.0, 0.0, 0, 0, n)], su2=su2_table([us]))


def rx_layer(state, beta: float) -> None:
    """exp(-i beta sum_q X_q) (reference mixers.py:87-91)."""
    n = num_qubits(state)
    with _OnDevice(state) as psi:
        run_program(psi, n, "x", [(0.0, beta, 0, 0, n)])


def apply_xy(state, beta: float, i: int, j: int) -> None:
    """exp(-i beta (X_i X_j + Y_i Y_j)/2) in place (reference mixers.py:94-106)."""
    n = num_qubits(state)
    if i == j:
        raise ValueError(f"XY coupling needs two distinct qubits, got ({i}, {j})")
    if not (0 <= i < n and 0 <= j < n):
        raise ValueError(f"pair ({i}, {j}) out of range for {n} qubits")
    with _OnDevice(state) as psi:
        _lib.call("fq_xy_on_pairs", psi.data_ptr(), psi.numel(), float(np.cos(beta)), float(np.sin(beta)),
                  min(i, j), max(i, j), _lib.stream())


def xy_ring_layer(state, beta: float) -> None:
    """reference mixers.py:128-131"""
    n = num_qubits(state)
    ring_edges(n)
    with _OnDevice(state) as psi:
        run_program(psi, n, "xy-ring", [(0.0, beta, 0, 0, n)])


def xy_complete_layer(state, beta: float) -> None:
    """reference mixers.py:134-137"""
    n = num_qubits(state)
    complete_edges(n)
    with _OnDevice(state) as psi:
        run_program(psi, n, "xy-complete", [(0.0, beta, 0, 0, n)])


class Mixer:
    """Per-layer mixing operator selected by kind (reference mixers.py:140-199):
    "x", "xy-ring", "xy-complete", or "custom" with an SU(2)-per-qubit factory."""

    KINDS = ("x", "xy-ring", "xy-complete", "custom")

    def __init__(self, kind: str, su2_factory: Callable[[float], Sequence[SU2]] | None = None) -> None:
        if kind not in self.KINDS:
            raise ValueError(f"unknown mixer kind {kind!r}; expected one of {self.KINDS}")
        if (kind == "custom") != (su2_factory is not None):
            raise ValueError("custom mixers take a factory; named mixers do not")
        self.kind = kind
        self.su2_factory = su2_factory

    @classmethod
    def x(cls) -> Mixer:
        return cls("x")

    @classmethod
    def xy_ring(cls) -> Mixer:
        return cls("xy-ring")

    @classmethod
    def xy_complete(cls) -> Mixer:
        return cls("xy-complete")

    @classmethod
    def custom(cls, su2_factory: Callable[[float], Sequence[SU2]]) -> Mixer:
        return cls("custom", su2_factory)

    @classmethod
    def parse(cls, value: "str | Mixer") -> Mixer:
        if isinstance(value, Mixer):
            return value
        return cls(value)

    @property
    def preserves_hamming_weight(self) -> bool:
        return self.kind in ("xy-ring", "xy-complete")

    def su2_table(self, betas: Sequence[float], n: int) -> np.ndarray | None:
        if self.kind != "custom":
            return None
        rows = []
        for b in betas:
            us = list(self.su2_factory(b))
            if len(us) != n:
                raise ValueError(f"expected {n} matrices, got {len(us)}")
            rows.append(us)
        if not rows:  # zero layers: a (never read) table keeps the descriptor valid
            return np.zeros((1, n, 4), dtype=np.float64)
        return su2_table(rows)

    def apply_layer(self, state, beta: float) -> None:
        if self.kind == "x":
            rx_layer(state, beta)
        elif self.kind == "xy-ring":
            xy_ring_layer(state, beta)
        elif self.kind == "xy-complete":
            xy_complete_layer(state, beta)
        else:
            apply_uniform_su2(state, self.su2_factory(beta))

    def __repr__(self) -> str:
        return f"Mixer({self.kind!r})"
