"""ctypes binding of libfqaoa.so (the C ABI declared in include/fqaoa.h).

The product path has exactly one implementation: the sm_100a kernels in
this library.  There is no CPU fallback — if the library or a CUDA device is
missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfqaoa.so")

FQ_OK, FQ_ERR_ARG, FQ_ERR_CUDA, FQ_ERR_UNSUPPORTED = 0, 1, 2, 3
FQ_SCRATCH_DOUBLES = 4096
MIXER_CODES = {"x": 0, "xy-ring": 1, "xy-complete": 2, "custom": 3}
COST_F64, COST_U16 = 0, 1
STATE_C128, STATE_C64 = 0, 1

P, I64, D, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int


class FqLayer(ctypes.Structure):
    _fields_ = [("gamma", D), ("beta", D), ("apply_phase", I), ("q_lo", I), ("q_hi", I)]


class FqEvolveDesc(ctypes.Structure):
    _fields_ = [
        ("psi", P), ("n", I), ("cost_kind", I), ("costs", P), ("cost_scale", D), ("cost_offset", D),
        ("cost_levels", I), ("mixer", I), ("n_layers", I), ("layers", ctypes.POINTER(FqLayer)), ("su2", ctypes.POINTER(D)),
        ("init", I), ("init_amp", D), ("expectation_dev", P), ("scratch", P), ("state_kind", I),
    ]


class FqShardDesc(ctypes.Structure):
    _fields_ = [
        ("k", I), ("rank", I), ("shards", ctypes.POINTER(P)), ("costs", ctypes.POINTER(P)),
        ("flags", ctypes.POINTER(P)), ("epoch", ctypes.POINTER(ctypes.c_uint)), ("barrier_err", P),
    ]


_SIGS = {
    "fq_version": ([], I),
    "fq_last_error": ([], ctypes.c_char_p),
    "fq_sm_count": ([], I),
    "fq_su2_on_pairs": ([P, I64, D, D, D, D, I, P], I),
    "fq_xy_on_pairs": ([P, I64, D, D, I, I, P], I),
    "fq_swap_bits": ([P, I64, I, I, P], I),
    "fq_phase_multiply": ([P, P, I64, D, P], I),
    "fq_accumulate_terms": ([P, I64, P, P, I64, I64, P], I),
    "fq_accumulate_terms_dyadic": ([P, I64, P, P, I64, I, I, I64, P], I),
    "fq_precompute_levels_u16": ([P, I64, P, P, I64, I, I64, I64, I, P, P], I),
    "fq_precompute_wht": ([P, I64, P, P, I64, I, I64, P], I),
    "fq_abs2_inplace": ([P, I64, P], I),
    "fq_init_state": ([P, I64, I, D, I64, P], I),
    "fq_expectation": ([P, P, I, D, D, I64, P, P, P], I),
    "fq_init_state_c64": ([P, I64, I, D, I64, P], I),
    "fq_abs2_inplace_c64": ([P, I64, P], I),
    "fq_expectation_c64": ([P, P, I, D, D, I64, P, P, P], I),
    "fq_masked_probability_c64": ([P, P, I, D, D, I64, D, P, P, P], I),
    "fq_cost_minmax": ([P, I, D, D, I64, P, P, P], I),
    "fq_masked_probability": ([P, P, I, D, D, I64, D, P, P, P], I),
    "fq_compact_u16": ([P, P, I64, D, D, P, P], I),
    "fq_rebase_u16": ([P, I64, I, P], I),
    "fq_qaoa_evolve": ([ctypes.POINTER(FqEvolveDesc), P], I),
    "fq_qaoa_objective": ([ctypes.POINTER(FqEvolveDesc), ctypes.POINTER(D), P], I),
    "fq_objective_graph_create": ([ctypes.POINTER(FqEvolveDesc), P, P, ctypes.POINTER(P)], I),
    "fq_objective_graph_run": ([P, P], I),
    "fq_objective_graph_destroy": ([P], I),
    "fq_qaoa_evolve_sharded": ([ctypes.POINTER(FqEvolveDesc), ctypes.POINTER(FqShardDesc), P], I),
    "fq_plan_sharded_passes": ([I, I, I, ctypes.POINTER(FqLayer), P], I),
    "fq_qaoa_evolve_batched": ([I, I, P, I, D, D, I, I, P, P, P, P, P, P], I),
    "fq_qaoa_evolve_batched_levels": ([I, I, P, I, D, D, I, I, I, P, P, P, P, P, P], I),
    "fq_plan_x_passes": ([I, I, ctypes.POINTER(FqLayer), I], I),
    "fq_set_option": ([ctypes.c_char_p, I], I),
    "fq_last_passes": ([P, P, I], I),
    "fq_plan_xy_passes": ([I, I, P], I),
    "fq_plan_x_describe": ([I, I, ctypes.POINTER(FqLayer), I, I, ctypes.c_char_p, I], I),
    "fq_global_su2_pass": ([P, I, I64, I, I, P, P], I),
    "fq_ipc_handle": ([P, P, P], I),
    "fq_ipc_open": ([P, I64, P], I),
    "fq_ipc_close": ([P, I64], I),
    "fq_peer_barrier": ([P, I, I, ctypes.c_uint, P, P], I),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load(path: str | None = None):
    """Load libfqaoa.so (no CUDA device needed to load).  FQ_LIB_VARIANT=<name>
    selects a development build of the same sources with other compile-time
    options (scripts/build_variant.py, A/B timing only); FQ_OPTIONS sets
    run-time options (fq_set_option) at load."""
    global _lib
    with _lock:
        if _lib is None:
            if path is None:
                var = os.environ.get("FQ_LIB_VARIANT")
                path = os.path.join(_HERE, "variants", var, "libfqaoa.so") if var else LIB_PATH
            if not os.path.exists(path):
                raise ImportError(
                    f"libfqaoa.so not found at {path}: build it with "
                    "`python -m paper_2309_04841_b200._build` (there is no CPU fallback)"
                )
            lib = ctypes.CDLL(path)
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
            # development: FQ_OPTIONS="name=value,..." applies fq_set_option at load
            # (A/B runs of the test suite under a kernel variant)
            for item in filter(None, os.environ.get("FQ_OPTIONS", "").split(",")):
                name, _, value = item.partition("=")
                if lib.fq_set_option(name.strip().encode(), int(value)) != FQ_OK:
                    raise ValueError(f"FQ_OPTIONS: {item}: {(lib.fq_last_error() or b'').decode()}")
    return _lib


def check(status: int, what: str = "") -> None:
    if status == FQ_OK:
        return
    msg = (load().fq_last_error() or b"").decode(errors="replace")
    if status == FQ_ERR_ARG:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: libfqaoa error {status}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


_cuda_ok = False  # a CUDA device was found once (it does not go away within a process)
_devices: dict[int, torch.device] = {}


def device() -> torch.device:
    """The CUDA device the simulator runs on; raises if none (no CPU fallback).
    On the path of every call: the availability probe runs once per process."""
    global _cuda_ok
    if not _cuda_ok:
        if not torch.cuda.is_available():
            raise RuntimeError(
                "paper_2309_04841_b200 needs a CUDA device (B200, sm_100a); "
                "there is no CPU fallback"
            )
        _cuda_ok = True
    idx = torch.cuda.current_device()
    dev = _devices.get(idx)
    if dev is None:
        dev = _devices[idx] = torch.device("cuda", idx)
    return dev


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream() -> int:
    """The caller's current CUDA stream (raw handle).  The direct C++ query costs
    ~0.3 us against ~3 us for torch.cuda.current_stream(): on the path of every
    small-n call."""
    if _raw_stream is not None:
        return _raw_stream(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


_scratch: dict[int, torch.Tensor] = {}


def scratch() -> torch.Tensor:
    idx = device().index
    buf = _scratch.get(idx)
    if buf is None:
        buf = torch.zeros(FQ_SCRATCH_DOUBLES, dtype=torch.float64, device=_devices[idx])
        _scratch[idx] = buf
    return buf


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def describe_x_plan(n: int, p: int, state_kind: int = STATE_C128, k: int = 0, phase: bool = True) -> str:
    """The X-mixer pass plan of a p-layer program over n qubits (k global):
    host-only (fq_plan_x_describe), e.g. for the planner tests."""
    lay = (FqLayer * max(1, p))(*[FqLayer(0.5 if phase else 0.0, 0.3, 1, 0, n) for _ in range(p)])
    buf = ctypes.create_string_buffer(8192)
    cnt = load().fq_plan_x_describe(n, p, lay, state_kind, k, buf, len(buf))
    if cnt < 0:
        raise ValueError(f"no X plan for n={n}, k={k}")
    return buf.value.decode()
