"""Layered QAOA evolution on a B200 (mirror of reference fastqaoa/qaoa.py).

The cost diagonal is evaluated once per problem on the GPU and stays
resident; ``simulate_qaoa`` enqueues one fused program (libfqaoa
``fq_qaoa_evolve``): phase and mixer layers batched 12 qubits per HBM pass,
with the objective sum c|psi|^2 folded into the last pass.  ``get_*``
accessors return host (CPU) values, as in the paper's API.
"""

from __future__ import annotations

import ctypes
import weakref
from collections import OrderedDict
from dataclasses import dataclass
from math import sqrt
from typing import Sequence

import numpy as np
import torch
from torch.autograd.graph import increment_version

from . import _lib, instrumentation
from .costs import DeviceCosts
from .mixers import Mixer, run_program
from .statevec import expectation_device, num_qubits, overlap_device
from .terms import TermPolynomial, _check_fits


@dataclass(frozen=True)
class QaoaParams:
    """Per-layer angle pairs (reference qaoa.py:31-60)."""

    gammas: tuple[float, ...]
    betas: tuple[float, ...]

    def __post_init__(self) -> None:
        object.__setattr__(self, "gammas", tuple(float(g) for g in self.gammas))
        object.__setattr__(self, "betas", tuple(float(b) for b in self.betas))
        if len(self.gammas) != len(self.betas):
            raise ValueError(f"{len(self.gammas)} gammas but {len(self.betas)} betas")

    @property
    def p(self) -> int:
        return len(self.gammas)

    @classmethod
    def from_flat(cls, x: Sequence[float]) -> QaoaParams:
        x = np.asarray(x, dtype=np.float64)
        if x.size % 2:
            raise ValueError(f"flat parameter vector has odd length {x.size}")
        p = x.size // 2
        return cls(tuple(x[:p]), tuple(x[p:]))

    def to_flat(self) -> np.ndarray:
        return np.array(self.gammas + self.betas, dtype=np.float64)


class QaoaResult:
    """Final state (device) plus the cost diagonal it was evolved under
    (reference qaoa.py:63-68).  ``state`` / ``costs`` are host numpy views
    copied on first access; ``state_device`` / ``costs_device`` stay on the GPU."""

    def __init__(self, state_device: torch.Tensor, costs_device: DeviceCosts,
                 expectation_dev: torch.Tensor | None = None):
        self.state_device = state_device
        self.costs_device = costs_device
        self._expectation_dev = expectation_dev
        self._state_host: np.ndarray | None = None
        # the state is live (reference qaoa.py:63-68): the library's in-place operations
        # bump its version counter (statevec._OnDevice), which retires the cached
        # objective of the fused last pass and the host copy
        self._version = state_device._version

    def _check_version(self) -> None:
        if self.state_device._version != self._version:
            self._mutated()
            self._version = self.state_device._version

    @property
    def state(self) -> np.ndarray:
        self._check_version()
        if self._state_host is None:
            self._state_host = self.state_device.cpu().numpy()
        return self._state_host

    def cached_expectation(self) -> torch.Tensor | None:
        """The objective computed by the program's last pass, if the state is unchanged since."""
        self._check_version()
        return self._expectation_dev

    @property
    def costs(self) -> np.ndarray:
        return self.costs_device.host()

    @property
    def n(self) -> int:
        return self.costs_device.n

    def _mutated(self) -> None:
        self._expectation_dev = None
        self._state_host = None


_COST_MEMO: "OrderedDict[TermPolynomial, DeviceCosts]" = OrderedDict()
_MEMO_SIZE = 32


def _device_costs_for(poly: TermPolynomial, state_bytes: int = 16) -> DeviceCosts:
    """Diagonal of a polynomial sized for one state of the same n next to it
    (``state_bytes`` per amplitude: 16 complex128, 8 complex64): float64 +
    uint16 levels when they fit, else (integer / dyadic weights, e.g. LABS
    n = 33 complex128 or n = 34 complex64 on one B200) the uint16 levels
    alone, computed exactly from the terms — the reference's n <= 30 cap
    (terms.py:109-113) becomes this device-memory check."""
    free, _ = torch.cuda.mem_get_info(_lib.device())
    size = 1 << poly.n
    if size * (state_bytes + 8 + 2) <= 0.95 * free:
        return DeviceCosts.from_polynomial(poly)
    if size * (state_bytes + 2) <= 0.95 * free:
        try:
            return DeviceCosts.from_polynomial(poly, keep_f64=False)
        except MemoryError:
            pass
    _check_fits(poly.n, state_bytes + 8, "state vector + cost vector")
    return DeviceCosts.from_polynomial(poly)


def _cached_device_costs(poly: TermPolynomial) -> DeviceCosts:
    """Process-wide memo of device diagonals (reference qaoa.py:71-75, lru 32)."""
    dc = _COST_MEMO.get(poly)
    if dc is not None:
        _COST_MEMO.move_to_end(poly)
        return dc
    _check_fits(poly.n, 2, "cost vector")
    dc = _device_costs_for(poly)
    instrumentation.bump("precompute")
    _COST_MEMO[poly] = dc
    while len(_COST_MEMO) > _MEMO_SIZE:
        _COST_MEMO.popitem(last=False)
    return dc


def resolve_costs(problem) -> tuple[DeviceCosts, int]:
    """Device diagonal + qubit count for a polynomial (memoised) or a ready
    2^n vector (reference qaoa.py:78-87)."""
    if isinstance(problem, TermPolynomial):
        return _cached_device_costs(problem), problem.n
    if isinstance(problem, DeviceCosts):
        return problem, problem.n
    dc = DeviceCosts.from_array(problem)
    return dc, dc.n


def state_dtype(dtype) -> torch.dtype:
    """complex128 (the reference's state, default) or complex64 (optional
    single-precision state; 1e-4 tolerance)."""
    if dtype is None:
        return torch.complex128
    if dtype in (torch.complex128, torch.complex64):
        return dtype
    name = np.dtype(dtype).name if not isinstance(dtype, str) else dtype
    if name in ("complex128", "c16", "complex"):
        return torch.complex128
    if name in ("complex64", "c8"):
        return torch.complex64
    raise ValueError(f"unsupported state dtype {dtype!r} (complex128 or complex64)")


def _initial_state(n: int, mixer: Mixer, initial, out: torch.Tensor | None = None,
                   dtype: torch.dtype = torch.complex128) -> tuple[torch.Tensor, bool]:
    """(device state, generate-|+>-in-kernel flag) — reference qaoa.py:90-103.
    ``out``: caller-owned buffer the |+> program evolves into (no allocation)."""
    dev = _lib.device()
    if initial is not None:
        if isinstance(initial, torch.Tensor):
            if initial.numel() != 1 << n:
                raise ValueError(f"initial state has {initial.numel()} amplitudes, expected {1 << n}")
            return initial.to(device=dev, dtype=dtype).clone().contiguous(), False
        arr = np.array(initial, dtype=np.complex128)
        if arr.size != 1 << n:
            raise ValueError(f"initial state has {arr.size} amplitudes, expected {1 << n}")
        return torch.from_numpy(arr.reshape(-1)).to(dev).to(dtype), False
    if mixer.preserves_hamming_weight:
        raise ValueError(
            "XY mixers act within a fixed-popcount sector; pass an initial "
            "state explicitly (see statevec.hamming_weight_state)"
        )
    if out is not None:
        return out, True
    try:
        return torch.empty(1 << n, dtype=dtype, device=dev), True
    except torch.OutOfMemoryError as exc:
        raise MemoryError(f"state vector for n={n} does not fit in device memory "
                          f"(shard it: simulate_qaoa_distributed / ShardedQaoaSimulator)") from exc


def _evolve(dc: DeviceCosts, n: int, mixer: Mixer, params: QaoaParams, initial,
            out: torch.Tensor | None = None, dtype: torch.dtype = torch.complex128) -> QaoaResult:
    if dtype == torch.complex64:
        if n <= 12:
            # on-chip sizes: the resident fp64 program, rounded to complex64 once at the end
            res = _evolve(dc, n, mixer, params, initial)
            return QaoaResult(res.state_device.to(torch.complex64), dc, res._expectation_dev)
    state, init = _initial_state(n, mixer, initial, out=out, dtype=dtype)
    layers = [(g, b, 1, 0, n) for g, b in zip(params.gammas, params.betas)]
    exp_dev = torch.empty(1, dtype=torch.float64, device=state.device)
    run_program(state, n, mixer.kind, layers, dc=dc, su2=mixer.su2_table(params.betas, n),
                init=init, init_amp=1.0 / sqrt(float(1 << n)), expectation_out=exp_dev)
    return QaoaResult(state, dc, exp_dev)


class _ObjectiveGraph:
    """A captured one-evaluation CUDA graph for n <= 12 (fq_objective_graph_*):
    pinned angle / objective buffers the kernel reads and writes directly, the
    graph handle, and references to the device buffers it uses (they must
    outlive it)."""

    def __init__(self, desc, p: int, state: torch.Tensor, exp_dev: torch.Tensor):
        self._ang_t = torch.empty(2 * p, dtype=torch.float64, pin_memory=True)
        self._out_t = torch.zeros(1, dtype=torch.float64, pin_memory=True)
        self.ang = self._ang_t.numpy()
        self._out = self._out_t.numpy()
        self._keep = (desc, state, exp_dev)
        h = ctypes.c_void_p()
        _lib.check(_lib.load().fq_objective_graph_create(ctypes.byref(desc), self._ang_t.data_ptr(),
                                                         self._out_t.data_ptr(), ctypes.byref(h)),
                   "fq_objective_graph_create")
        self._h = h
        self._finalizer = weakref.finalize(self, _lib.load().fq_objective_graph_destroy, h)

    def run(self) -> float:
        _lib.check(_lib.load().fq_objective_graph_run(self._h, _lib.stream()), "fq_objective_graph_run")
        return float(self._out[0])



class QaoaSimulator:
    """Simulator bound to one problem; the cost diagonal is computed once, on
    the GPU, at construction (reference qaoa.py:106-166)."""

    def __init__(self, n: int | None = None, *, terms=None, costs=None, mixer: "str | Mixer" = "x",
                 dtype=None) -> None:
        """``dtype``: state type, complex128 (default, the reference's) or
        complex64 (optional: half the HBM traffic and memory, every mixer,
        amplitudes / objective within 1e-4 of complex128)."""
        if (terms is None) == (costs is None):
            raise ValueError("pass exactly one of terms= or costs=")
        self.dtype = state_dtype(dtype)
        if terms is not None:
            if not isinstance(terms, TermPolynomial):
                if n is None:
                    raise ValueError("a plain term list needs n")
                terms = TermPolynomial.from_pairs(n, terms)
            _check_fits(terms.n, 2, "cost vector")
            self._dc = _device_costs_for(terms, state_bytes=16 if self.dtype == torch.complex128 else 8)
            instrumentation.bump("precompute")
            self.n = terms.n
        else:
            self._dc = costs if isinstance(costs, DeviceCosts) else DeviceCosts.from_array(costs)
            self.n = self._dc.n
        if n is not None and n != self.n:
            raise ValueError(f"n={n} disagrees with problem size {self.n}")
        self.mixer = Mixer.parse(mixer)
        self._buffer: torch.Tensor | None = None
        self._obj_ctx = None  # objective(): prepared descriptor for the last depth
        self._graph_ctx = None  # objective(), n <= 12: captured CUDA graph for the last depth

    @property
    def device_costs(self) -> DeviceCosts:
        return self._dc

    def get_cost_diagonal(self) -> np.ndarray:
        return self._dc.host()

    def simulate_qaoa(self, gammas: Sequence[float], betas: Sequence[float], initial=None,
                      reuse_buffer: bool = False) -> QaoaResult:
        """Run the layered evolution; the result's state lives on the GPU.

        ``reuse_buffer=True`` evolves into one simulator-owned state buffer
        (objective loops at large n: no per-call allocation; the previous
        result's state is overwritten)."""
        params = QaoaParams(tuple(gammas), tuple(betas))
        out = None
        if reuse_buffer:
            if self._buffer is None:
                self._buffer = torch.empty(1 << self.n, dtype=self.dtype, device=_lib.device())
            out = self._buffer
        return _evolve(self._dc, self.n, self.mixer, params, initial, out=out, dtype=self.dtype)

    use_graph = True  # objective() for n <= 12: replay a captured CUDA graph (fq_objective_graph_*)

    def objective(self, gammas: Sequence[float], betas: Sequence[float], initial=None) -> float:
        """<C> of one parameter set — the optimiser-loop call (reference
        qaoa_objective, qaoa.py:185-194, bound to this simulator): the
        evolution runs in the simulator-owned state buffer and the objective
        comes from the program's last pass; one host synchronisation.  X mixer
        from |+>: one prepared descriptor per depth, one ABI call per
        evaluation (fq_qaoa_objective: program, copy-out, synchronise)."""
        if initial is not None or self.mixer.kind != "x":
            res = self.simulate_qaoa(gammas, betas, initial=initial, reuse_buffer=True)
            return float(res.cached_expectation().item())
        gctx = self._graph_ctx
        if gctx is not None and self.use_graph and gctx[0] == len(gammas) == len(betas):
            # small states (n <= 12): replay the captured graph of this depth -- the
            # kernel reads the angles from this pinned array and writes the objective
            # into pinned memory (fq_objective_graph_run)
            og = gctx[1]
            og.ang[0::2] = gammas
            og.ang[1::2] = betas
            val = og.run()
            increment_version(self._buffer)
            return val
        gs, bs = tuple(float(g) for g in gammas), tuple(float(b) for b in betas)
        if len(gs) != len(bs):
            raise ValueError(f"{len(gs)} gammas but {len(bs)} betas")
        ctx = self._obj_ctx
        if ctx is None or ctx[0] != len(gs) or self._buffer is None:
            if self._buffer is None:
                self._buffer = torch.empty(1 << self.n, dtype=self.dtype, device=_lib.device())
            p = len(gs)
            arr = (_lib.FqLayer * max(1, p))()
            exp_dev = torch.empty(1, dtype=torch.float64, device=self._buffer.device)
            desc = _lib.FqEvolveDesc()
            desc.psi = self._buffer.data_ptr()
            desc.n = self.n
            kind, cp, scale, offset = self._dc.kernel_view()
            desc.cost_kind, desc.costs, desc.cost_scale, desc.cost_offset = kind, cp, scale, offset
            desc.cost_levels = self._dc.levels if kind == _lib.COST_U16 else 0
            desc.mixer = _lib.MIXER_CODES["x"]
            desc.n_layers = p
            desc.layers = arr
            desc.init = 1
            desc.init_amp = 1.0 / sqrt(float(1 << self.n))
            desc.expectation_dev = exp_dev.data_ptr()
            desc.scratch = _lib.scratch().data_ptr()
            desc.state_kind = _lib.STATE_C64 if self.dtype == torch.complex64 else _lib.STATE_C128
            ctx = self._obj_ctx = (p, arr, desc, exp_dev, ctypes.c_double(), _lib.load().fq_qaoa_objective)
        _, arr, desc, _, out, fn = ctx
        for i, (g, b) in enumerate(zip(gs, bs)):
            L = arr[i]
            L.gamma, L.beta, L.apply_phase, L.q_lo, L.q_hi = g, b, 1, 0, self.n
        if self.n <= 12 and self.dtype == torch.complex128 and self.use_graph and len(gs) <= 64:
            # first evaluation at this depth: capture the graph, then replay it (above)
            self._graph_ctx = (len(gs), _ObjectiveGraph(desc, len(gs), self._buffer, ctx[3]))
            return self.objective(gs, bs)
        _lib.check(fn(ctypes.byref(desc), ctypes.byref(out), _lib.stream()), "fq_qaoa_objective")
        increment_version(self._buffer)  # a reuse_buffer result's state was overwritten
        return out.value

    def simulate_qaoa_batched(self, gammas, betas) -> np.ndarray:
        """Expectations of many parameter sets at once (n <= 12: each set
        runs in its own CTA, one launch).  gammas, betas: [batch, p]."""
        g = np.ascontiguousarray(gammas, dtype=np.float64)
        b = np.ascontiguousarray(betas, dtype=np.float64)
        if g.ndim != 2 or g.shape != b.shape:
            raise ValueError("gammas and betas must both be [batch, p]")
        if self.n > 12 or self.mixer.kind == "custom" or self.dtype == torch.complex64:
            return np.array([self.get_expectation(self.simulate_qaoa(gg, bb)) for gg, bb in zip(g, b)])
        if self.mixer.preserves_hamming_weight:
            raise ValueError("XY mixers need an explicit initial state; use simulate_qaoa")
        batch, p = g.shape
        out = torch.empty(batch, dtype=torch.float64, device=_lib.device())
        kind, cp, scale, offset = self._dc.kernel_view()
        chunk = max(1, 512 // max(p, 1))
        for s in range(0, batch, chunk):
            e = min(batch, s + chunk)
            gs, bs = np.ascontiguousarray(g[s:e]), np.ascontiguousarray(b[s:e])
            levels = self._dc.levels if kind == _lib.COST_U16 else 0
            _lib.call("fq_qaoa_evolve_batched_levels", self.n, _lib.MIXER_CODES[self.mixer.kind], cp, kind, scale,
                      offset, levels, p, e - s, gs.ctypes.data, bs.ctypes.data, None, None, out[s:].data_ptr(), _lib.stream())
        return out.cpu().numpy()

    def get_statevector(self, result: QaoaResult) -> np.ndarray:
        return result.state

    def get_probabilities(self, result: QaoaResult, preserve_state: bool = True) -> np.ndarray:
        """|psi|^2 as a host array (reference qaoa.py:154, statevec.py:81-91).
        ``preserve_state=False`` squares the result's state in place and returns
        the real view of that state, as the reference does: the result's state
        then holds |psi|^2 + 0j (on the device and in ``result.state``)."""
        psi = result.state_device
        work = psi.clone() if preserve_state else psi
        fn = "fq_abs2_inplace_c64" if work.dtype == torch.complex64 else "fq_abs2_inplace"
        _lib.call(fn, work.data_ptr(), work.numel(), _lib.stream())
        if preserve_state:
            return torch.view_as_real(work)[:, 0].cpu().numpy()
        increment_version(psi)
        result._mutated()
        return result.state.real  # a view of the (now squared) state, like state.real in the reference

    def get_expectation(self, result: QaoaResult, costs=None) -> float:
        if costs is None:
            cached = result.cached_expectation()
            if cached is not None:
                return float(cached.item())
            dc = result.costs_device
        else:
            dc = costs if isinstance(costs, DeviceCosts) else DeviceCosts.from_array(costs, compact=False)
            if dc.size != result.state_device.numel():
                raise ValueError(
                    f"state has {result.state_device.numel()} amplitudes but cost vector has {dc.size} entries")
        return float(expectation_device(result.state_device, dc).item())

    def get_overlap(self, result: QaoaResult, costs=None, tol: float = 0.0) -> float:
        if costs is None:
            dc = result.costs_device
        else:
            dc = costs if isinstance(costs, DeviceCosts) else DeviceCosts.from_array(costs, compact=False)
            if dc.size != result.state_device.numel():
                raise ValueError(
                    f"state has {result.state_device.numel()} amplitudes but cost vector has {dc.size} entries")
        lo, _ = dc.minmax()
        total = float(overlap_device(result.state_device, dc, lo + tol).item())
        return min(max(total, 0.0), 1.0)


def simulate_qaoa(problem, params: QaoaParams, mixer: "str | Mixer" = "x", initial=None,
                  dtype=None) -> QaoaResult:
    """One-shot evolution; the device diagonal is memoised per polynomial
    (reference qaoa.py:169-182).  ``dtype``: see QaoaSimulator."""
    dc, n = resolve_costs(problem)
    return _evolve(dc, n, Mixer.parse(mixer), params, initial, dtype=state_dtype(dtype))


def qaoa_objective(problem, params: QaoaParams, mixer: "str | Mixer" = "x", initial=None, dtype=None) -> float:
    """Expected cost of the evolved state (reference qaoa.py:185-194)."""
    result = simulate_qaoa(problem, params, mixer=mixer, initial=initial, dtype=dtype)
    return float(result.cached_expectation().item())


__all__ = ["QaoaParams", "QaoaResult", "QaoaSimulator", "simulate_qaoa", "qaoa_objective", "resolve_costs",
           "num_qubits", "state_dtype"]
