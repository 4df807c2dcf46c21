"""TEST INFRASTRUCTURE ONLY — CPU oracle for the QAOA hot path.

A restatement of the reference's algorithm (fastqaoa, /root/reference/pkg)
on top of the plain-C kernels in ``fqaoa_oracle.c``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
(``cpu_baseline`` / ``--impl reference``) may import this module, and only as
the checker or as the timed CPU baseline.  The product package
``paper_2309_04841_b200`` never imports it.

Parity pin: ``tests/test_oracle_golden.py`` compares every function here with
vectors produced by the reference itself (``scripts/gen_golden.py`` imports
``/root/reference/pkg/src``; fixtures in ``tests/golden/``).

Conventions (reference ``statevec.py:3-4``, ``terms.py:4-5``): qubit q is bit
q of the index; spin s_q = 1 - 2*bit_q.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from math import comb, sqrt

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None


def build() -> str:
    """Compile the oracle library (gcc + OpenMP) if missing or stale."""
    src = os.path.join(_HERE, "fqaoa_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P, I64, D, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        L.or_su2_on_pairs.argtypes = [P, I64, D, D, D, D, I]
        L.or_xy_on_pairs.argtypes = [P, I64, D, D, I, I]
        L.or_swap_bits.argtypes = [P, I64, I, I]
        L.or_phase_multiply.argtypes = [P, P, I64, D]
        L.or_accumulate_terms.argtypes = [P, I64, P, P, I64, I64]
        L.or_abs2_inplace.argtypes = [P, I64]
        L.or_expectation.argtypes = [P, P, I64]
        L.or_expectation.restype = D
        L.or_num_threads.restype = I
        for f in ("or_su2_on_pairs", "or_xy_on_pairs", "or_swap_bits",
                  "or_phase_multiply", "or_accumulate_terms", "or_abs2_inplace"):
            getattr(L, f).restype = None
        _lib = L
    return _lib


def num_threads() -> int:
    return int(lib().or_num_threads())


def _c128(a: np.ndarray) -> np.ndarray:
    assert a.dtype == np.complex128 and a.flags.c_contiguous
    return a


# ---------------------------------------------------------------- kernels
def su2_on_pairs(psi, a: complex, b: complex, q: int) -> None:
    """reference _kernels.py:14-27"""
    _c128(psi)
    lib().or_su2_on_pairs(psi.ctypes.data, psi.size, a.real, a.imag, b.real, b.imag, q)


def xy_on_pairs(psi, cos_b: float, sin_b: float, p_lo: int, p_hi: int) -> None:
    """reference _kernels.py:30-48"""
    _c128(psi)
    lib().or_xy_on_pairs(psi.ctypes.data, psi.size, cos_b, sin_b, p_lo, p_hi)


def swap_bits(psi, p_lo: int, p_hi: int) -> None:
    """reference _kernels.py:51-65"""
    _c128(psi)
    lib().or_swap_bits(psi.ctypes.data, psi.size, p_lo, p_hi)


def phase_multiply(psi, costs, gamma: float) -> None:
    """reference _kernels.py:68-73"""
    _c128(psi)
    costs = np.ascontiguousarray(costs, dtype=np.float64)
    lib().or_phase_multiply(psi.ctypes.data, costs.ctypes.data, psi.size, gamma)


def accumulate_terms(out, weights, masks, base: int = 0) -> None:
    """reference _kernels.py:76-94 (``base`` = global index of out[0])."""
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    masks = np.ascontiguousarray(masks, dtype=np.int64)
    lib().or_accumulate_terms(out.ctypes.data, out.size, weights.ctypes.data,
                              masks.ctypes.data, weights.size, base)


def abs2_inplace(psi) -> None:
    """reference _kernels.py:97-102"""
    _c128(psi)
    lib().or_abs2_inplace(psi.ctypes.data, psi.size)


# ---------------------------------------------------------------- operators
def terms_arrays(terms):
    """(weights f64[T], masks int64[T]) — reference terms.py:116-117.

    ``terms`` is a sequence of (weight, support) pairs."""
    weights = np.array([float(w) for w, _ in terms], dtype=np.float64)
    masks = np.array([sum(1 << int(i) for i in s) for _, s in terms], dtype=np.int64)
    return weights, masks


def precompute_cost_vector(n: int, terms, base: int = 0, size: int | None = None) -> np.ndarray:
    """reference terms.py:102-120 (without the n<=30 guard: a shard of
    ``size`` entries starting at global index ``base`` can be evaluated)."""
    size = (1 << n) if size is None else size
    values = np.zeros(size)
    if len(terms):
        w, m = terms_arrays(terms)
        accumulate_terms(values, w, m, base)
    return values


def uniform_state(n: int) -> np.ndarray:
    """reference statevec.py:22-29"""
    dim = 1 << n
    return np.full(dim, 1.0 / sqrt(dim), dtype=np.complex128)


def hamming_weight_state(n: int, weight: int) -> np.ndarray:
    """reference statevec.py:41-54"""
    state = np.zeros(1 << n, dtype=np.complex128)
    idx = np.flatnonzero(np.bitwise_count(np.arange(1 << n, dtype=np.uint64)) == weight)
    state[idx] = 1.0 / sqrt(comb(n, weight))
    return state


def apply_phase(state, costs, gamma: float) -> None:
    """reference statevec.py:69-78 (gamma == 0 is a bit-exact no-op)."""
    if gamma == 0.0:
        return
    phase_multiply(state, costs, gamma)


def rx_coeffs(beta: float):
    """SU2.rx — reference mixers.py:47-50: (cos b, -i sin b)."""
    from cmath import cos, sin
    return complex(cos(beta)), -1j * sin(beta)


def rx_layer(state, beta: float) -> None:
    """reference mixers.py:87-91 (ascending qubit sweep)."""
    a, b = rx_coeffs(beta)
    n = state.size.bit_length() - 1
    for q in range(n):
        su2_on_pairs(state, a, b, q)


def apply_uniform_su2(state, us) -> None:
    """reference mixers.py:74-84; ``us`` = [(a, b)] per qubit."""
    for q, (a, b) in enumerate(us):
        su2_on_pairs(state, complex(a), complex(b), q)


def ring_edges(n: int):
    """reference mixers.py:109-118"""
    if n == 2:
        return [(0, 1)]
    edges = [(q, q + 1) for q in range(0, n - 1, 2)]
    edges += [(q, q + 1) for q in range(1, n - 1, 2)]
    edges.append((n - 1, 0))
    return edges


def complete_edges(n: int):
    """reference mixers.py:121-125"""
    return [(i, j) for i in range(n) for j in range(i + 1, n)]


def apply_xy(state, beta: float, i: int, j: int) -> None:
    """reference mixers.py:94-106"""
    xy_on_pairs(state, float(np.cos(beta)), float(np.sin(beta)), min(i, j), max(i, j))


def mixer_layer(state, kind: str, beta: float, su2_factory=None) -> None:
    """reference mixers.py:188-196"""
    n = state.size.bit_length() - 1
    if kind == "x":
        rx_layer(state, beta)
    elif kind == "xy-ring":
        for i, j in ring_edges(n):
            apply_xy(state, beta, i, j)
    elif kind == "xy-complete":
        for i, j in complete_edges(n):
            apply_xy(state, beta, i, j)
    elif kind == "custom":
        apply_uniform_su2(state, su2_factory(beta))
    else:
        raise ValueError(kind)


def simulate(costs, gammas, betas, kind: str = "x", initial=None, su2_factory=None) -> np.ndarray:
    """QaoaSimulator.simulate_qaoa loop — reference qaoa.py:137-149:
    per layer, phase then mixer."""
    n = costs.size.bit_length() - 1
    state = uniform_state(n) if initial is None else np.array(initial, dtype=np.complex128)
    for g, b in zip(gammas, betas):
        apply_phase(state, costs, float(g))
        mixer_layer(state, kind, float(b), su2_factory)
    return state


def probabilities(state) -> np.ndarray:
    """reference statevec.py:81-91 (preserve_state=True)."""
    return np.abs(state) ** 2


def expectation(state, costs) -> float:
    """reference statevec.py:94-97"""
    return float(np.dot(costs, probabilities(state)))


def expectation_fast(state, costs) -> float:
    """Same quantity with the C/OpenMP reduction (CPU baseline timing)."""
    _c128(state)
    costs = np.ascontiguousarray(costs, dtype=np.float64)
    return float(lib().or_expectation(state.ctypes.data, costs.ctypes.data, state.size))


def overlap(state, costs, tol: float = 0.0) -> float:
    """reference statevec.py:100-111"""
    ground = costs <= costs.min() + tol
    return min(max(float(np.sum(np.abs(state[ground]) ** 2)), 0.0), 1.0)


# ---------------------------------------------------------------- sharding
def exchange(shards):
    """all_to_all_exchange — reference distributed.py:103-122: subchunk j of
    worker i swaps with subchunk i of worker j (V[a,b,c] -> V[b,a,c])."""
    K = len(shards)
    sub = shards[0].size // K
    mailbox = [[shards[i][j * sub:(j + 1) * sub].copy() for i in range(K)] for j in range(K)]
    for i in range(K):
        for j in range(K):
            shards[i][j * sub:(j + 1) * sub] = mailbox[i][j]


def transpose_oracle(state, k: int) -> np.ndarray:
    """Index formula for the exchange (reference tests/test_distributed.py:25-37)."""
    n = state.size.bit_length() - 1
    V = state.reshape(1 << k, 1 << k, 1 << (n - 2 * k))
    return np.ascontiguousarray(V.transpose(1, 0, 2)).reshape(-1)


# ---------------------------------------------------------------- problems
def labs_terms(n: int):
    """reference problems.py:128-146 — (weight, support) pairs, same order."""
    terms = []
    for i in range(1, n - 2):
        for t in range(1, (n - i - 1) // 2 + 1):
            for k in range(t + 1, n - i - t + 1):
                terms.append((2.0, (i - 1, i + t - 1, i + k - 1, i + k + t - 1)))
    for i in range(1, n - 1):
        for k in range(1, (n - i) // 2 + 1):
            terms.append((1.0, (i - 1, i + 2 * k - 1)))
    return terms


def labs_energy(k: int, n: int) -> int:
    """reference problems.py:149-163 (independent oracle)."""
    bits = (k >> np.arange(n)) & 1
    spins = 1 - 2 * bits
    return int(sum(int(np.dot(spins[: n - t], spins[t:])) ** 2 for t in range(1, n)))
