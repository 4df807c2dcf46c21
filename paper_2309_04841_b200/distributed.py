"""State sharding by global qubits (mirror of reference fastqaoa/distributed.py).

Worker r owns global indices [r 2^(n-k), (r+1) 2^(n-k)) — the top k index
bits are the "global" qubits (reference distributed.py:1-23, 51-54).  The
only collective is the subchunk all-to-all V[a,b,c] -> V[b,a,c]
(distributed.py:103-122): after it the former global qubits sit at local
positions n-2k .. n-k-1, so an X-mixer layer is: local passes, exchange,
one pass over k positions, exchange (Alg. 4).

Two deployments of the same orchestration:

* ``simulate_qaoa_distributed`` / ``ShardedState`` — K logical workers
  inside one process on one GPU (the reference's own model, same API and
  exchange counters); the exchange is a device transpose.
* ``ShardedQaoaSimulator`` — one process per GPU (torchrun), shard-local
  precompute by index offset (no n<=30 cap), exchange = NCCL all-to-all over
  NVLink (``torch.distributed.all_to_all_single``, ncclAlltoAll), scalar
  reductions = ``all_reduce``.  Local work is always libfqaoa.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from math import comb, sqrt
from typing import Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import _lib, instrumentation
from .costs import DeviceCosts
from .mixers import SU2, Mixer, complete_edges, ring_edges, run_program, su2_table
from .qaoa import QaoaParams, QaoaResult, _initial_state, resolve_costs, state_dtype
from .statevec import expectation_device, overlap_device
from .terms import TermPolynomial


def _validate_split(n: int, K: int) -> int:
    """K = 2^k with 2k <= n (reference distributed.py:39-48; messages are test-matched)."""
    k = K.bit_length() - 1
    if K < 1 or (1 << k) != K:
        raise ValueError(f"worker count {K} is not a power of two")
    if 2 * k > n:
        raise ValueError(
            f"{K} workers split {n} qubits into subchunks smaller than one "
            f"amplitude (need 2*log2(K) <= n)"
        )
    return k


# ====================================================================== in-process
@dataclass
class ShardedState:
    """K = 2^k shards of one state (reference distributed.py:51-62).  On the
    device all shards are views of one [K, 2^(n-k)] buffer."""

    n: int
    k: int
    shards: list
    exchange_count: int = 0

    @property
    def K(self) -> int:
        return 1 << self.k


@dataclass
class ShardedCosts:
    """Cost diagonal sliced like the state (reference distributed.py:65-72)."""

    n: int
    k: int
    shards: list


def _as_device_vector(x) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=_lib.device()).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x)).to(_lib.device())


def scatter(state, K: int) -> ShardedState:
    """Split into K private shards (reference distributed.py:75-85)."""
    size = state.numel() if isinstance(state, torch.Tensor) else np.asarray(state).size
    n = (size - 1).bit_length()
    if size != 1 << n:
        raise ValueError(f"state length {size} is not a power of two")
    k = _validate_split(n, K)
    buf = _as_device_vector(np.asarray(state, dtype=np.complex128) if not isinstance(state, torch.Tensor) else state)
    buf = buf.to(torch.complex128).clone().view(K, 1 << (n - k))
    return ShardedState(n, k, list(buf.unbind(0)))


def gather(sharded: ShardedState) -> np.ndarray:
    """Concatenated host state (reference distributed.py:88-89)."""
    return torch.cat([s.reshape(-1) for s in sharded.shards]).cpu().numpy()


def shard_costs(costs, K: int) -> ShardedCosts:
    """Slice a cost vector like the state (reference distributed.py:92-100)."""
    if isinstance(costs, DeviceCosts):
        n = costs.n
        k = _validate_split(n, K)
        return ShardedCosts(n, k, _slice_device_costs(costs, K))
    arr = np.asarray(costs, dtype=np.float64)
    n = (arr.size - 1).bit_length()
    if arr.size != 1 << n:
        raise ValueError(f"cost length {arr.size} is not a power of two")
    k = _validate_split(n, K)
    return ShardedCosts(n, k, _slice_device_costs(DeviceCosts.from_array(arr), K))


def _slice_device_costs(dc: DeviceCosts, K: int) -> list[DeviceCosts]:
    n_local = dc.n - (K.bit_length() - 1)
    size = 1 << n_local
    out = []
    for r in range(K):
        f = dc.f64[r * size:(r + 1) * size] if dc.f64 is not None else None
        u = dc.u16[r * size:(r + 1) * size] if dc.u16 is not None else None
        out.append(DeviceCosts(n_local, f64=f, u16=u, scale=dc.scale, offset=dc.offset, levels=dc.levels))
    return out


def all_to_all_exchange(sharded: ShardedState) -> None:
    """Subchunk j of worker i <-> subchunk i of worker j, in place; self-inverse
    (reference distributed.py:103-122).  One device transpose of V[K,K,sub]."""
    K = sharded.K
    sub = 1 << (sharded.n - 2 * sharded.k)
    V = torch.stack([s.reshape(K, sub) for s in sharded.shards])  # [a, b, c]
    T = V.transpose(0, 1).contiguous()                             # [b, a, c]
    for a in range(K):
        sharded.shards[a].copy_(T[a].reshape(-1))
    sharded.exchange_count += 1
    instrumentation.bump("exchange")


def _check_slicing(sharded: ShardedState, costs: ShardedCosts) -> None:
    if (costs.n, costs.k) != (sharded.n, sharded.k):
        raise ValueError("cost slicing does not match the state slicing")


def apply_phase_distributed(sharded: ShardedState, costs: ShardedCosts, gamma: float) -> None:
    """Per-shard phase, no communication (reference distributed.py:125-134)."""
    _check_slicing(sharded, costs)
    if gamma == 0.0:
        return
    n_local = sharded.n - sharded.k
    for shard, dc in zip(sharded.shards, costs.shards):
        run_program(shard, n_local, "x", [(gamma, 0.0, 1, 0, 0)], dc=dc)


def _local_su2(sharded: ShardedState, us: Sequence[SU2], positions: range, offset: int) -> None:
    """Apply us[pos + offset] at local positions ``positions`` on every shard."""
    n_local = sharded.n - sharded.k
    table = [SU2.identity()] * n_local
    for pos in positions:
        table[pos] = us[pos + offset]
    t = su2_table([table])
    for shard in sharded.shards:
        run_program(shard, n_local, "custom", [(0.0, 0.0, 0, positions.start, positions.stop)], su2=t)


def apply_uniform_su2_distributed(sharded: ShardedState, us: Sequence[SU2]) -> None:
    """Local qubits, exchange, former global qubits at q-k, exchange — exactly
    two exchanges (reference distributed.py:137-153)."""
    n, k = sharded.n, sharded.k
    if len(us) != n:
        raise ValueError(f"expected {n} matrices, got {len(us)}")
    _local_su2(sharded, us, range(0, n - k), 0)
    all_to_all_exchange(sharded)
    _local_su2(sharded, us, range(n - 2 * k, n - k), k)
    all_to_all_exchange(sharded)


def rx_layer_distributed(sharded: ShardedState, beta: float) -> None:
    apply_uniform_su2_distributed(sharded, [SU2.rx(beta)] * sharded.n)


def _xy_local(sharded: ShardedState, beta: float, lo: int, hi: int) -> None:
    c, s = float(np.cos(beta)), float(np.sin(beta))
    for shard in sharded.shards:
        _lib.call("fq_xy_on_pairs", shard.data_ptr(), shard.numel(), c, s, lo, hi, _lib.stream())


def _swap_local(sharded: ShardedState, lo: int, hi: int) -> None:
    for shard in sharded.shards:
        _lib.call("fq_swap_bits", shard.data_ptr(), shard.numel(), lo, hi, _lib.stream())


def apply_xy_distributed(sharded: ShardedState, beta: float, i: int, j: int) -> None:
    """XY gate on a sharded state (reference distributed.py:160-207): local
    pairs directly; pairs touching a global qubit inside an exchange pair,
    parking a subchunk-id partner at position 0 with swap_bits."""
    n, k = sharded.n, sharded.k
    if i == j:
        raise ValueError(f"XY coupling needs two distinct qubits, got ({i}, {j})")
    if not (0 <= i < n and 0 <= j < n):
        raise ValueError(f"pair ({i}, {j}) out of range for {n} qubits")
    lo, hi = min(i, j), max(i, j)
    n_local = n - k
    if hi < n_local:
        _xy_local(sharded, beta, lo, hi)
        return
    b_start = n - 2 * k
    parked = False
    if b_start <= lo < n_local:
        if b_start == 0:
            raise ValueError(
                f"pair ({i}, {j}) spans the subchunk-id and worker-id qubits; "
                f"with 2*log2(K) == n there is no local position to stage it "
                f"(use fewer workers)"
            )
        _swap_local(sharded, 0, lo)
        lo, parked = 0, True
    pos_lo = lo - k if lo >= n_local else lo
    pos_hi = hi - k
    all_to_all_exchange(sharded)
    _xy_local(sharded, beta, min(pos_lo, pos_hi), max(pos_lo, pos_hi))
    all_to_all_exchange(sharded)
    if parked:
        _swap_local(sharded, 0, min(i, j))


def _mixer_layer_distributed(sharded: ShardedState, mixer: Mixer, beta: float) -> None:
    if mixer.kind == "x":
        rx_layer_distributed(sharded, beta)
    elif mixer.kind in ("xy-ring", "xy-complete"):
        edges = ring_edges(sharded.n) if mixer.kind == "xy-ring" else complete_edges(sharded.n)
        for i, j in edges:
            apply_xy_distributed(sharded, beta, i, j)
    else:
        apply_uniform_su2_distributed(sharded, mixer.su2_factory(beta))


def expectation_distributed(sharded: ShardedState, costs: ShardedCosts) -> float:
    """Sum of per-shard partials (reference distributed.py:228-237)."""
    _check_slicing(sharded, costs)
    parts = [expectation_device(s, c) for s, c in zip(sharded.shards, costs.shards)]
    return float(torch.cat(parts).cpu().numpy().sum())


def overlap_distributed(sharded: ShardedState, costs: ShardedCosts, tol: float = 0.0) -> float:
    """Global min, masked sum, clamp (reference distributed.py:240-252)."""
    _check_slicing(sharded, costs)
    cutoff = min(c.minmax()[0] for c in costs.shards) + tol
    parts = [overlap_device(s, c, cutoff) for s, c in zip(sharded.shards, costs.shards)]
    return min(max(float(torch.cat(parts).cpu().numpy().sum()), 0.0), 1.0)


@dataclass
class DistributedResult:
    """Evolved sharded state + sliced diagonal (reference distributed.py:255-277)."""

    sharded: ShardedState
    sharded_costs: ShardedCosts
    costs_device: DeviceCosts = field(repr=False)

    @property
    def exchange_count(self) -> int:
        return self.sharded.exchange_count

    @property
    def costs(self) -> np.ndarray:
        return self.costs_device.host()

    def statevector(self) -> np.ndarray:
        return gather(self.sharded)

    def expectation(self) -> float:
        return expectation_distributed(self.sharded, self.sharded_costs)

    def overlap(self, tol: float = 0.0) -> float:
        return overlap_distributed(self.sharded, self.sharded_costs, tol=tol)

    def to_result(self) -> QaoaResult:
        state = torch.cat([s.reshape(-1) for s in self.sharded.shards]).clone()
        return QaoaResult(state, self.costs_device)


def global_su2_pass(shard_ptrs: Sequence[int], k: int, shard_size: int, part: int, parts: int,
                    us: Sequence[SU2]) -> None:
    """libfqaoa fq_global_su2_pass: u_j on global qubit j across the 2^k peer-mapped
    shards, in place, for local indices of `part` of `parts`."""
    import ctypes

    ptrs = (ctypes.c_void_p * len(shard_ptrs))(*shard_ptrs)
    coef = np.array([(complex(u.a).real, complex(u.a).imag, complex(u.b).real, complex(u.b).imag) for u in us],
                    dtype=np.float64)
    _lib.call("fq_global_su2_pass", ptrs, k, shard_size, part, parts, coef.ctypes.data, _lib.stream())


def cost_consensus(allv, mine):
    """One cost encoding for all shards of a fused sharded program.

    ``allv[r]`` = (has_u16, has_f64, scale, offset, top) of rank r's shard
    (top = decoded value of its highest level); ``mine`` = this rank's.
    Returns (kind, offset, levels, delta): uint16 when every shard has
    levels on one scale and the union range fits 16 bits — the common origin
    is the global minimum and this rank's levels move up by ``delta`` — else
    float64 (then every shard must have kept it)."""
    if all(v[0] for v in allv) and len({v[2] for v in allv}) == 1:
        scale = allv[0][2]
        lo = min(v[3] for v in allv)
        hi = max(v[4] for v in allv)
        levels = int(round((hi - lo) / scale)) + 1
        if levels <= 65536:
            return _lib.COST_U16, lo, levels, int(round((mine[3] - lo) / scale))
    if not all(v[1] for v in allv):
        raise MemoryError("sharded cost encodings disagree and the float64 diagonal was not kept "
                          "(use global_mode='p2p' or 'exchange')")
    return _lib.COST_F64, 0.0, 0, 0


def _logical_exchanges(mixer: Mixer, n: int, k: int, p: int) -> int:
    """The reference's exchange count for p layers (API contract): Alg. 4's two
    per X / custom layer, two per gate touching a global qubit for XY mixers
    (distributed.py:160-207)."""
    if mixer.kind in ("x", "custom"):
        return 2 * p
    edges = ring_edges(n) if mixer.kind == "xy-ring" else complete_edges(n)
    return 2 * p * sum(1 for i, j in edges if max(i, j) >= n - k)


def evolve_sharded(shard_ptrs: Sequence[int], cost_ptrs: Sequence[int], costs: DeviceCosts, n: int, k: int,
                   mixer: Mixer, params: QaoaParams, init: bool, rank: int = -1, flags=None, epoch=None,
                   err_ptr: int | None = None, expectation_out: torch.Tensor | None = None,
                   dtype: torch.dtype = torch.complex128) -> None:
    """libfqaoa fq_qaoa_evolve_sharded: the whole p-layer program on a state
    sharded by its top k qubits — local groups as passes on each shard, the
    global group as peer-memory passes over all shards, fused across layers.
    ``rank`` -1: every shard is this process's (one stream, no barriers);
    else this rank's shard plus the peer barrier (``flags``, ``epoch``, ``err_ptr``)."""
    K = 1 << k
    nl = n - k
    dc = costs
    arr = (_lib.FqLayer * max(1, params.p))(*[_lib.FqLayer(float(g), float(b), 1, 0, n)
                                              for g, b in zip(params.gammas, params.betas)])
    desc = _lib.FqEvolveDesc()
    desc.n = nl
    if dc.u16 is not None:
        desc.cost_kind, desc.cost_scale, desc.cost_offset, desc.cost_levels = _lib.COST_U16, dc.scale, dc.offset, dc.levels
    else:
        desc.cost_kind, desc.cost_scale, desc.cost_offset, desc.cost_levels = _lib.COST_F64, 1.0, 0.0, 0
    desc.mixer = _lib.MIXER_CODES[mixer.kind]
    desc.n_layers = params.p
    desc.layers = arr
    su2 = mixer.su2_table(params.betas, n) if mixer.kind == "custom" else None
    su2_keep = None
    if su2 is not None:
        su2_keep = np.ascontiguousarray(su2, dtype=np.float64)
        desc.su2 = su2_keep.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    desc.init = 1 if init else 0
    desc.init_amp = 1.0 / sqrt(float(2 ** n)) if init else 0.0
    desc.expectation_dev = expectation_out.data_ptr() if expectation_out is not None else None
    desc.scratch = _lib.scratch().data_ptr()
    desc.state_kind = _lib.STATE_C64 if dtype == torch.complex64 else _lib.STATE_C128
    sd = _lib.FqShardDesc()
    sd.k = k
    sd.rank = rank
    shards = (ctypes.c_void_p * K)(*shard_ptrs)
    cps = (ctypes.c_void_p * K)(*cost_ptrs)
    sd.shards, sd.costs = shards, cps
    if rank >= 0:
        fl = (ctypes.c_void_p * K)(*flags)
        sd.flags = fl
        sd.epoch = ctypes.pointer(epoch)
        sd.barrier_err = err_ptr
    _lib.check(_lib.load().fq_qaoa_evolve_sharded(ctypes.byref(desc), ctypes.byref(sd), _lib.stream()),
               "fq_qaoa_evolve_sharded")
    del su2_keep


def simulate_qaoa_distributed(problem, params: QaoaParams, K: int, mixer: "str | Mixer" = "x",
                              initial=None, fused: bool = True, dtype=None) -> DistributedResult:
    """K logical workers on the current GPU (reference distributed.py:280-296).
    For the X mixer, phase + local qubits run as one fused program per shard;
    the global qubits run in one peer-memory pass over all shards (``fused``;
    False = the reference's exchange -> pass -> exchange)."""
    dc, n = resolve_costs(problem)
    mixer = Mixer.parse(mixer)
    k = _validate_split(n, K)
    dtype = state_dtype(dtype)
    if dtype == torch.complex64 and not (fused and 1 <= k <= 3 and n - k >= 12 and mixer.kind != "custom"):
        raise ValueError("complex64 sharded states run the fused program: X / XY mixers, K = 2..8, "
                         ">= 12 qubits per shard")
    state, init = _initial_state(n, mixer, initial, dtype=dtype)
    if init and dtype == torch.complex64:
        init_fn = "fq_init_state_c64"
    else:
        init_fn = "fq_init_state"
    if init:
        _lib.call(init_fn, state.data_ptr(), state.numel(), -1, 1.0 / sqrt(float(1 << n)), 0, _lib.stream())
    sharded = ShardedState(n, k, list(state.view(K, -1).unbind(0)))
    sc = ShardedCosts(n, k, _slice_device_costs(dc, K))
    n_local = n - k
    if fused and 1 <= k <= 3 and n_local >= 12:
        # one sharded program: the global group's passes span the K shard views
        # (the same kernels a multi-GPU rank runs over peer memory)
        cost_t = [c.u16 if c.u16 is not None else c.f64 for c in sc.shards]
        evolve_sharded([s.data_ptr() for s in sharded.shards], [t.data_ptr() for t in cost_t], sc.shards[0], n, k,
                       mixer, params, init, rank=-1, dtype=dtype)
        ex = _logical_exchanges(mixer, n, k, params.p)  # the reference's logical count
        sharded.exchange_count += ex
        instrumentation.bump("exchange", ex)
        return DistributedResult(sharded, sc, dc)
    for gamma, beta in zip(params.gammas, params.betas):
        if mixer.kind == "custom" and k > 0 and fused and k <= 4:
            us = list(mixer.su2_factory(beta))
            if len(us) != n:
                raise ValueError(f"expected {n} matrices, got {len(us)}")
            table = su2_table([us[:n_local]])
            for shard, c in zip(sharded.shards, sc.shards):
                run_program(shard, n_local, "custom", [(gamma, beta, 1, 0, n_local)], dc=c, su2=table)
            global_su2_pass([s.data_ptr() for s in sharded.shards], k, 1 << n_local, 0, 1, us[n_local:])
            sharded.exchange_count += 2
            instrumentation.bump("exchange", 2)
            continue
        if mixer.kind == "x" and k > 0:
            for shard, c in zip(sharded.shards, sc.shards):
                run_program(shard, n_local, "x", [(gamma, beta, 1, 0, n_local)], dc=c)
            if fused and k <= 4:
                # one peer-memory kernel replaces exchange -> k-position pass -> exchange;
                # the two logical exchanges of Alg. 4 are still counted (reference API)
                global_su2_pass([s.data_ptr() for s in sharded.shards], k, 1 << n_local, 0, 1, [SU2.rx(beta)] * k)
                sharded.exchange_count += 2
                instrumentation.bump("exchange", 2)
                continue
            all_to_all_exchange(sharded)
            for shard in sharded.shards:
                run_program(shard, n_local, "x", [(0.0, beta, 0, n_local - k, n_local)])
            all_to_all_exchange(sharded)
        else:
            apply_phase_distributed(sharded, sc, gamma)
            _mixer_layer_distributed(sharded, mixer, beta)
    return DistributedResult(sharded, sc, dc)


# ====================================================================== one process per GPU
class ShardedQaoaSimulator:
    """One rank per GPU; this rank holds global indices
    [rank 2^(n-k), (rank+1) 2^(n-k)).  Launch with torchrun; the process
    group must be NCCL for CUDA shards.

    Per X layer (Alg. 4): [phase + local qubits] fused passes, NCCL all-to-all,
    one pass over the k former-global positions, NCCL all-to-all.  The
    exchange double-buffers (receive into a second shard buffer, then swap
    pointers) when memory allows, else runs in bounded chunks."""

    def __init__(self, poly: TermPolynomial, group=None, mixer: "str | Mixer" = "x",
                 compact: bool = True, keep_f64: bool | None = None, chunk_bytes: int | None = None,
                 local_ops=None, global_mode: str | None = None, device_barrier: bool = True, dtype=None):
        """``global_mode`` (how mixer gates on the k global qubits run):
        "fused" (default on CUDA ranks with >= 12 local qubits) — one sharded
        program whose global-group passes span every shard over peer memory;
        "p2p" — a per-layer peer-memory kernel (the default below 12 local
        qubits); "exchange" — the reference's NCCL all-to-all structure (the
        default with custom ``local_ops``, e.g. the CPU test backend).
        ``dtype``: complex128 (default) or complex64 (global_mode="fused",
        X / XY mixers: half the memory per rank, e.g. n = 35 on two B200s)."""
        self.group = group
        self.dtype = state_dtype(dtype)
        self.K = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n = poly.n
        self.k = _validate_split(self.n, self.K)
        self.n_local = self.n - self.k
        self.mixer = Mixer.parse(mixer)
        if global_mode is None:
            global_mode = ("exchange" if local_ops is not None or self.k == 0
                           else "fused" if self.n_local >= 12 else "p2p")
        if self.dtype == torch.complex64 and (global_mode != "fused" or self.mixer.kind == "custom" or self.k == 0):
            raise ValueError("complex64 sharded states need global_mode='fused', the X or XY mixers and >= 2 ranks")
        self.ops = local_ops if local_ops is not None else CudaLocalOps()
        base = self.rank << self.n_local
        if keep_f64 is None:
            keep_f64 = self.ops.fits(self.n_local, 8 + (8 + 2 if self.dtype == torch.complex64 else 16 * 2 + 2))
        self.costs = self.ops.precompute(poly, base, self.n_local, compact, keep_f64)
        instrumentation.bump("precompute")
        self.exchange_count = 0
        self.chunk_bytes = chunk_bytes
        self._state = None
        self._spare = None
        if global_mode not in ("exchange", "p2p", "fused"):
            raise ValueError(f"global_mode must be 'exchange', 'p2p' or 'fused', got {global_mode!r}")
        self.global_mode = global_mode
        self.device_barrier = device_barrier
        self._p2p_buf = None
        self._peers: list[int] | None = None
        self._flag_ptrs: list[int] | None = None
        self._cost_peers: list[int] | None = None
        self._opened: list[tuple[int, int]] = []
        self._epoch = ctypes.c_uint(0)
        self._broken: str | None = None
        if global_mode == "fused" and self.k > 0:
            self._common_cost_encoding()

    # ------------------------------------------------------------------ exchange
    def exchange(self, shard: torch.Tensor) -> torch.Tensor:
        """V[a,b,c] -> V[b,a,c] across ranks; returns the tensor now holding the shard."""
        K = self.K
        if K == 1:
            return shard
        full_ok = self.chunk_bytes is None and (self._spare is not None or self.ops.fits_bytes(shard.numel() * 16))
        if full_ok:
            if self._spare is None or self._spare.numel() != shard.numel():
                self._spare = torch.empty_like(shard)
            self._a2a(self._spare, shard)
            out, self._spare = self._spare, shard
        else:
            # bounded staging: column block [c0, c1) of every subchunk per round;
            # row j of the send block goes to rank j, row a of the receive
            # block came from rank a, i.e. V_me[a, c] = V_a[me, c].
            sub = shard.numel() // K
            V = shard.view(K, sub)
            piece = max(1, min(sub, (self.chunk_bytes or (256 << 20)) // (16 * K)))
            for c0 in range(0, sub, piece):
                c1 = min(sub, c0 + piece)
                send = V[:, c0:c1].contiguous()
                recv = torch.empty_like(send)
                self._a2a(recv, send)
                V[:, c0:c1].copy_(recv)
            out = shard
        self.exchange_count += 1
        instrumentation.bump("exchange")
        return out

    def _a2a(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        """all_to_all_single; over a CPU-only backend (gloo) CUDA shards are
        staged through host memory (NCCL moves them GPU to GPU over NVLink)."""
        if inp.is_cuda and dist.get_backend(self.group) == "gloo":
            host = torch.empty_like(inp, device="cpu")
            dist.all_to_all_single(host, inp.cpu(), group=self.group)
            out.copy_(host)
        else:
            dist.all_to_all_single(out, inp, group=self.group)

    # ------------------------------------------------------------------ evolution
    def initial_state(self, initial_weight: int | None = None) -> torch.Tensor:
        if initial_weight is None:
            return self.ops.uniform(self.n, self.n_local)
        return self.ops.hamming(self.n, initial_weight, self.rank << self.n_local, self.n_local)

    def simulate_qaoa(self, gammas: Sequence[float], betas: Sequence[float], initial_weight: int | None = None,
                      expectation: bool = True) -> float | None:
        """Evolve; returns the global expectation (all-reduced) if requested."""
        if self._broken:
            raise RuntimeError(self._broken)
        params = QaoaParams(tuple(gammas), tuple(betas))
        if self.mixer.preserves_hamming_weight and initial_weight is None:
            raise ValueError("XY mixers need initial_weight (Hamming-weight sector)")
        if self.mixer.preserves_hamming_weight:
            return self._simulate_xy(params, initial_weight, expectation)
        nl, k = self.n_local, self.k
        if self.global_mode == "fused" and k > 0:
            return self._simulate_fused(params, initial_weight, expectation)
        if self.global_mode == "p2p" and k > 0:
            psi = self._p2p_shard()
            if initial_weight is not None:
                psi.copy_(self.initial_state(initial_weight))
        else:
            psi = self.ops.empty(nl) if initial_weight is None else self.initial_state(initial_weight)
        init = initial_weight is None
        amp = 1.0 / sqrt(float(2 ** self.n)) if init else 0.0
        custom = self.mixer.kind == "custom"
        for li, (g, b) in enumerate(zip(params.gammas, params.betas)):
            us = None
            if custom:
                us = list(self.mixer.su2_factory(b))
                if len(us) != self.n:
                    raise ValueError(f"expected {self.n} matrices, got {len(us)}")
            self.ops.program(psi, nl, self.mixer.kind, [(g, b, 1, 0, nl)], self.costs, init=init and li == 0,
                             init_amp=amp, su2=su2_table([us[:nl]]) if custom else None)
            glob = us[nl:] if custom else [SU2.rx(b)] * k
            if k > 0 and self.global_mode == "p2p":
                self._global_p2p(glob)
            elif k > 0:
                psi = self.exchange(psi)
                if custom:  # former global qubit n-k+j sits at local position nl-k+j (Alg. 4)
                    table = [SU2.identity()] * (nl - k) + glob
                    self.ops.program(psi, nl, "custom", [(0.0, b, 0, nl - k, nl)], None, su2=su2_table([table]))
                else:
                    self.ops.program(psi, nl, "x", [(0.0, b, 0, nl - k, nl)], None)
                psi = self.exchange(psi)
        if params.p == 0 and init:
            psi = self.ops.uniform(self.n, nl)
        self._state = psi
        if not expectation:
            return None
        return self.expectation()

    # ------------------------------------------------------------------ peer-memory global pass
    def _p2p_shard(self) -> torch.Tensor:
        """Persistent shard buffer, mapped into every rank (CUDA IPC handles
        all-gathered once).  NVLink peers on one node; on one device (tests)
        the same IPC path maps another process's allocation."""
        if self._p2p_buf is None:
            self._p2p_buf = (torch.empty(1 << self.n_local, dtype=torch.complex64, device=_lib.device())
                             if self.dtype == torch.complex64 else self.ops.empty(self.n_local))
            # flag arrays of the device-side barrier (K uint32 slots per rank) + error word
            self._flags = torch.zeros(self.K + 1, dtype=torch.int32, device=self._p2p_buf.device)
            torch.cuda.synchronize()  # zeroed before any peer can store into it
            self._peers = self._map_peers(self._p2p_buf.data_ptr())
            self._flag_ptrs = self._map_peers(self._flags.data_ptr())
        return self._p2p_buf

    def _map_peers(self, ptr: int) -> list[int]:
        """All-gather the CUDA IPC handle of a local buffer; map every peer's."""
        h = (ctypes.c_char * 64)()
        off = ctypes.c_int64()
        _lib.call("fq_ipc_handle", ptr, h, ctypes.byref(off))
        allh = [None] * self.K
        dist.all_gather_object(allh, (bytes(h), off.value), group=self.group)
        out = []
        for r, (hb, o) in enumerate(allh):
            if r == self.rank:
                out.append(ptr)
                continue
            p = ctypes.c_void_p()
            _lib.call("fq_ipc_open", hb, o, ctypes.byref(p))
            out.append(p.value)
            self._opened.append((p.value, o))
        return out

    def _barrier(self) -> None:
        """Order this rank's stream against every rank's: a stream-ordered
        flag barrier in peer memory (fq_peer_barrier, no host sync), or host
        synchronisation + dist.barrier."""
        if self.device_barrier:
            self._epoch.value += 1
            ptrs = (ctypes.c_void_p * self.K)(*self._flag_ptrs)
            _lib.call("fq_peer_barrier", ptrs, self.K, self.rank, self._epoch.value,
                      self._flags.data_ptr() + 4 * self.K, _lib.stream())
        else:
            torch.cuda.synchronize()
            dist.barrier(group=self.group)

    def check_barrier(self) -> None:
        """Raise if a device-side peer barrier timed out (host sync).  Runs
        after every peer-memory program, whatever it returns.  After a timeout
        the shards' contents are undefined (passes may have raced a rank that
        never arrived): the error word is cleared and the simulator refuses
        further work instead of computing on them."""
        if self._broken:
            raise RuntimeError(self._broken)
        if self._p2p_buf is not None and self.device_barrier and int(self._flags[self.K].item()) != 0:
            self._flags[self.K].zero_()
            self._broken = ("peer barrier timed out (a rank did not arrive); the sharded state is undefined — "
                            "create a new ShardedQaoaSimulator")
            raise RuntimeError(self._broken)

    def _global_p2p(self, us: Sequence[SU2]) -> None:
        """Alg. 4's exchange -> k-position pass -> exchange as ONE peer-memory
        kernel per rank (fq_global_su2_pass): rank r transforms the local
        indices of its 1/K part across all K shards, in place.  Two barriers
        order it against every rank's local passes.  Logical exchange count
        as in the reference (2 per layer)."""
        self._barrier()
        global_su2_pass(self._peers, self.k, 1 << self.n_local, self.rank, self.K, us)
        self._barrier()
        self.exchange_count += 2
        instrumentation.bump("exchange", 2)

    # ------------------------------------------------------------------ fused sharded program
    def _common_cost_encoding(self) -> None:
        """Peer-memory passes decode any shard's costs with one (scale,
        offset): uint16 shards agree on the scale and move to the global
        minimum as origin (fq_rebase_u16), else every shard uses float64."""
        dc = self.costs
        mine = (dc.u16 is not None, dc.f64 is not None, dc.scale, dc.offset,
                dc.offset + (dc.levels - 1) * dc.scale if dc.u16 is not None else 0.0)
        allv = [None] * self.K
        dist.all_gather_object(allv, mine, group=self.group)
        kind, offset, levels, delta = cost_consensus(allv, mine)
        self._cost_kind = kind
        if kind == _lib.COST_U16:
            if delta:
                _lib.call("fq_rebase_u16", dc.u16.data_ptr(), dc.u16.numel(), -delta, _lib.stream())
            dc.offset = offset
            dc.levels = levels

    def _cost_tensor(self) -> torch.Tensor:
        return self.costs.u16 if self._cost_kind == _lib.COST_U16 else self.costs.f64

    def _simulate_fused(self, params: QaoaParams, initial_weight, expectation: bool):
        """One fq_qaoa_evolve_sharded program: local groups on this shard,
        the global group as peer-memory passes fused across layers."""
        n, nl, K = self.n, self.n_local, self.K
        if nl < 12:
            raise ValueError(f"global_mode='fused' needs >= 12 qubits per shard (got {nl}); use 'p2p'")
        psi = self._p2p_shard()
        if self._cost_peers is None:
            self._cost_peers = self._map_peers(self._cost_tensor().data_ptr())
        init = initial_weight is None
        if not init:
            psi.copy_(self.initial_state(initial_weight))
        exp = torch.zeros(1, dtype=torch.float64, device=psi.device) if expectation else None
        view = DeviceCosts(nl, u16=self.costs.u16, scale=self.costs.scale, offset=self.costs.offset,
                           levels=self.costs.levels) if self._cost_kind == _lib.COST_U16 else \
            DeviceCosts(nl, f64=self.costs.f64)
        evolve_sharded(self._peers, self._cost_peers, view, n, self.k, self.mixer, params, init, rank=self.rank,
                       flags=self._flag_ptrs, epoch=self._epoch, err_ptr=self._flags.data_ptr() + 4 * K,
                       expectation_out=exp, dtype=self.dtype)
        # the reference's logical exchange count (Alg. 4: two per X layer)
        ex = _logical_exchanges(self.mixer, n, self.k, params.p)
        self.exchange_count += ex
        instrumentation.bump("exchange", ex)
        self._state = psi
        if not expectation:
            self.check_barrier()  # mandatory after every peer-memory program
            return None
        # one host synchronisation: the objective's partial sums and every rank's
        # barrier error word are all-reduced together
        out = torch.stack([exp[0], self._flags[K].to(torch.float64)])
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=self.group)
        e, err = out.tolist()
        if err != 0.0:
            self._flags[K].zero_()
            self._broken = ("peer barrier timed out on some rank (a rank did not arrive); the sharded state is "
                            "undefined — create a new ShardedQaoaSimulator")
            raise RuntimeError(self._broken)
        return e

    def close(self) -> None:
        for ptr, off in self._opened:
            _lib.call("fq_ipc_close", ptr, off)
        self._opened = []
        self._peers = None

    # ------------------------------------------------------------------ XY mixers
    def _xy_gate(self, psi: torch.Tensor, beta: float, i: int, j: int) -> torch.Tensor:
        """One XY gate on the sharded state (reference distributed.py:160-207):
        local pairs directly; a pair touching a global qubit inside an
        exchange pair, a subchunk-id partner parked at local position 0."""
        n, k, nl = self.n, self.k, self.n_local
        lo, hi = min(i, j), max(i, j)
        if hi < nl:
            self.ops.xy(psi, beta, lo, hi)
            return psi
        b_start = n - 2 * k
        parked = False
        if b_start <= lo < nl:
            if b_start == 0:
                raise ValueError(
                    f"pair ({i}, {j}) spans the subchunk-id and worker-id qubits; "
                    f"with 2*log2(K) == n there is no local position to stage it (use fewer workers)"
                )
            self.ops.swap(psi, 0, lo)
            lo, parked = 0, True
        pos_lo = lo - k if lo >= nl else lo
        pos_hi = hi - k
        psi = self.exchange(psi)
        self.ops.xy(psi, beta, min(pos_lo, pos_hi), max(pos_lo, pos_hi))
        psi = self.exchange(psi)
        if parked:
            self.ops.swap(psi, 0, min(i, j))
        return psi

    def _simulate_xy(self, params: QaoaParams, initial_weight: int, expectation: bool):
        nl = self.n_local
        if self.global_mode == "fused" and self.k > 0 and nl >= 12:
            return self._simulate_fused(params, initial_weight, expectation)
        edges = ring_edges(self.n) if self.mixer.kind == "xy-ring" else complete_edges(self.n)
        psi = self.initial_state(initial_weight)
        for g, b in zip(params.gammas, params.betas):
            if g != 0.0:
                self.ops.program(psi, nl, "x", [(g, 0.0, 1, 0, 0)], self.costs)
            for i, j in edges:
                psi = self._xy_gate(psi, b, i, j)
        self._state = psi
        return self.expectation() if expectation else None

    def expectation(self) -> float:
        self.check_barrier()
        local = self.ops.expectation(self._state, self.costs)
        dist.all_reduce(local, op=dist.ReduceOp.SUM, group=self.group)
        return float(local.item())

    def statevector(self) -> np.ndarray:
        """The full state on every rank (the reference's DistributedResult.statevector
        = gather of the shards, distributed.py:267-268); only for sizes that fit
        one host.  Collective: every rank must call it.  Refuses (MemoryError)
        when the gathered vector would not fit this host's free memory — e.g.
        n = 34 complex128 is 256 GiB; stream shards with ``save_shard`` instead."""
        self.check_barrier()
        t = self._state
        need = t.numel() * t.element_size() * self.K
        if need > _host_free_bytes():
            raise MemoryError(f"statevector(): the gathered {self.n}-qubit state needs {need / 2**30:.1f} GiB of host "
                              f"memory ({_host_free_bytes() / 2**30:.1f} GiB free); use save_shard() per rank")
        if t.is_cuda and dist.get_backend(self.group) == "gloo":
            t = t.cpu()
        t = t.contiguous()
        parts = [torch.empty_like(t) for _ in range(self.K)]
        dist.all_gather(parts, t, group=self.group)
        return torch.cat(parts).cpu().numpy()

    def save_shard(self, path: str, chunk_bytes: int = 256 << 20) -> None:
        """Stream this rank's shard to ``path`` in bounded device->host chunks
        (little-endian interleaved complex, the layout of statevec.save_state;
        shard r holds global indices [r 2^(n-k), (r+1) 2^(n-k))).  Concatenating
        the K files in rank order gives the reference's save_state file of the
        whole state (statevec.py:114-117) — the egress path for states that
        do not fit one host."""
        self.check_barrier()
        t = self._state.reshape(-1)
        step = max(1, chunk_bytes // t.element_size())
        pinned = torch.empty(min(step, t.numel()), dtype=t.dtype, pin_memory=t.is_cuda)
        with open(path, "wb") as f:
            for s0 in range(0, t.numel(), step):
                s1 = min(t.numel(), s0 + step)
                buf = pinned[:s1 - s0]
                buf.copy_(t[s0:s1])
                f.write(buf.numpy().astype("<c16" if t.dtype == torch.complex128 else "<c8", copy=False).tobytes())

    def overlap(self, tol: float = 0.0) -> float:
        lo = self.ops.min_cost(self.costs)
        dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=self.group)
        part = self.ops.masked_probability(self._state, self.costs, float(lo.item()) + tol)
        dist.all_reduce(part, op=dist.ReduceOp.SUM, group=self.group)
        return min(max(float(part.item()), 0.0), 1.0)

    @property
    def shard(self) -> torch.Tensor:
        return self._state


def _host_free_bytes() -> int:
    try:
        import psutil

        return int(psutil.virtual_memory().available)
    except Exception:  # noqa: BLE001 - no psutil: assume the gather fits
        return 1 << 62


class CudaLocalOps:
    """Shard-local work for ShardedQaoaSimulator: always libfqaoa on the
    rank's CUDA device (no fallback)."""

    def fits(self, n_local: int, bytes_per_amp: int) -> bool:
        free, _ = torch.cuda.mem_get_info(_lib.device())
        return (1 << n_local) * bytes_per_amp < 0.9 * free

    def fits_bytes(self, nbytes: int) -> bool:
        free, _ = torch.cuda.mem_get_info(_lib.device())
        return nbytes < 0.9 * free

    def precompute(self, poly, base: int, n_local: int, compact: bool, keep_f64: bool) -> DeviceCosts:
        return DeviceCosts.from_polynomial(poly, compact=compact, keep_f64=keep_f64, index_base=base,
                                           n_local=n_local)

    def empty(self, n_local: int) -> torch.Tensor:
        return torch.empty(1 << n_local, dtype=torch.complex128, device=_lib.device())

    def uniform(self, n: int, n_local: int) -> torch.Tensor:
        psi = self.empty(n_local)
        _lib.call("fq_init_state", psi.data_ptr(), psi.numel(), -1, 1.0 / sqrt(float(2 ** n)), 0, _lib.stream())
        return psi

    def hamming(self, n: int, weight: int, base: int, n_local: int) -> torch.Tensor:
        psi = self.empty(n_local)
        _lib.call("fq_init_state", psi.data_ptr(), psi.numel(), weight, 1.0 / sqrt(comb(n, weight)), base,
                  _lib.stream())
        return psi

    def program(self, psi, n_local, kind, layers, costs, init=False, init_amp=0.0, su2=None):
        run_program(psi, n_local, kind, layers, dc=costs, su2=su2, init=init, init_amp=init_amp)

    def xy(self, psi, beta, lo, hi):
        _lib.call("fq_xy_on_pairs", psi.data_ptr(), psi.numel(), float(np.cos(beta)), float(np.sin(beta)), lo, hi,
                  _lib.stream())

    def swap(self, psi, lo, hi):
        _lib.call("fq_swap_bits", psi.data_ptr(), psi.numel(), lo, hi, _lib.stream())

    def expectation(self, psi, costs) -> torch.Tensor:
        return expectation_device(psi, costs)

    def min_cost(self, costs) -> torch.Tensor:
        return torch.tensor([costs.minmax()[0]], dtype=torch.float64, device=_lib.device())

    def masked_probability(self, psi, costs, cutoff) -> torch.Tensor:
        return overlap_device(psi, costs, cutoff)


__all__ = [
    "ShardedState", "ShardedCosts", "scatter", "gather", "shard_costs", "all_to_all_exchange",
    "apply_phase_distributed", "apply_uniform_su2_distributed", "rx_layer_distributed", "apply_xy_distributed",
    "expectation_distributed", "overlap_distributed", "DistributedResult", "simulate_qaoa_distributed",
    "ShardedQaoaSimulator", "CudaLocalOps",
]
