"""Benchmark: QAOA objective evaluations/s for LABS (n=26, p=10, complex128) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n N] [--p P]

One "step" = one full QAOA objective evaluation: |+>^n -> p x (phase, X mixer)
-> sum_k c_k |psi_k|^2 (BASELINE.json north star, LABS n=26 p=10 fp64).

* ``value``: device-resident throughput (cost diagonal resident in HBM, the
  fused program enqueued back to back, CUDA events on the launching stream).
  The 1 GiB state is ~8x the 126 MB L2, so no L2 flush is needed between steps.
* ``e2e``: the same metric through the public API a user calls —
  ``sim.simulate_qaoa(gammas, betas)`` + ``sim.get_expectation(result)`` —
  angles from host memory each step (fresh values), the scalar read back.
* ``roofline``: HBM bound of the dominant kernel (k_tile_pass); achieved =
  algorithmic bytes of the step's tile passes / their time.
* ``cpu_baseline``: the CPU oracle port (oracle/, C + OpenMP restatement of the
  reference's numba kernels) on this host, bounded sample.
* N > 1 (torchrun): the state is sharded by global qubits, weak scaling with
  n = 26 + log2 N (2^26 amplitudes per GPU); exchanges are NCCL all-to-all.
  ``value`` counts n=26-equivalent evaluations (one n-qubit evaluation =
  2^(n-26) of them) so ideal weak scaling is N x the 1-GPU value.
* ``--impl reference``: the reference algorithm's CPU implementation (the
  oracle port; the reference is Python/numba, there is nothing to compile)
  on all host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASE_N = 26
PASS_NAMES = {-1: "phase sweep", 0: "8|0|4", 1: "8|4", 2: "8|0|4|0|8", 3: "8|4|8"}


def pass_name(sq: int) -> str:
    """Round program of a pass record; >= 100: an L2 slab sweep of two passes."""
    if sq >= 100:
        return f"sweep[{PASS_NAMES[(sq - 100) // 10]} > {PASS_NAMES[(sq - 100) % 10]}]"
    return PASS_NAMES.get(sq, str(sq))
METRIC = "QAOA objective evals/sec (LABS/MaxCut n=26–34); achieved HBM GB/s vs peak"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def angles(p, seed=0):
    rng = np.random.default_rng(seed)
    return rng.uniform(0, 1, p), rng.uniform(0, 1, p)


class ClockSampler:
    """Samples SM clocks + throttle reasons via NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()
        return False

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        reasons = [name for bit, name in self.REASONS.items() if self.reasons & bit and bit != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------- CPU (oracle port)
def cpu_eval_rate(costs, p, g, b, layers_sample):
    """Time `layers_sample` QAOA layers + one expectation with the oracle
    (C + OpenMP), extrapolate to a p-layer evaluation."""
    from oracle import oracle as O

    n = costs.size.bit_length() - 1
    st = O.uniform_state(n)
    t0 = time.perf_counter()
    for li in range(layers_sample):
        O.apply_phase(st, costs, float(g[li % p]))
        O.rx_layer(st, float(b[li % p]))
    t_layers = (time.perf_counter() - t0) / layers_sample
    t0 = time.perf_counter()
    O.expectation_fast(st, costs)
    t_exp = time.perf_counter() - t0
    t_eval = p * t_layers + t_exp
    return 1.0 / t_eval, t_layers, t_exp


def cpu_model() -> str:
    """Host CPU model (for the CPU baseline's provenance)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, rank):
    if rank != 0:
        return
    from oracle import oracle as O

    n = args.n or BASE_N
    p = args.p
    g, b = angles(p)
    threads = O.num_threads()
    t0 = time.perf_counter()
    costs = O.precompute_cost_vector(n, O.labs_terms(n))
    t_pre = time.perf_counter() - t0
    st = O.uniform_state(n)
    # one step = one QAOA layer (phase + X mixer over all n qubits) of the
    # p-layer evaluation; the objective rate combines p layers + 1 expectation.
    for w in range(args.warmup):
        O.apply_phase(st, costs, float(g[w % p]))
        O.rx_layer(st, float(b[w % p]))
    t0 = time.perf_counter()
    for s in range(args.steps):
        O.apply_phase(st, costs, float(g[s % p]))
        O.rx_layer(st, float(b[s % p]))
    t_layer = (time.perf_counter() - t0) / args.steps
    t0 = time.perf_counter()
    O.expectation_fast(st, costs)
    t_exp = time.perf_counter() - t0
    value = 1.0 / (p * t_layer + t_exp)
    sample = (f"{args.steps} timed layers (phase + X mixer) of LABS n={n}; evals/s = 1/(p*t_layer + t_expectation), "
              f"p={p}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_layer, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": f"LABS n={n} p={p} X-mixer complex128 objective evaluation", "n": n, "p": p,
                   "step": "one QAOA layer", "l2": "state > L2"},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "port", "sample": sample,
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "precompute_s": t_pre, "ms_per_layer": 1e3 * t_layer, "ms_expectation": 1e3 * t_exp,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- extra BASELINE configs
def S_total_bytes(n, c64):
    """Bytes of one n-qubit state."""
    return (8 if c64 else 16) << n


def _event_ms(fn, reps, world):
    """Device time of `reps` calls, CUDA events on the current stream, max over ranks."""
    import torch
    import torch.distributed as dist

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def run_config3(args):
    """BASELINE config 3: LABS n=30 p=10 objective inside a COBYLA loop (scipy),
    precompute once; evals/s including every evaluation's host round trip
    (the optimiser's own time included), next to the reference algorithm's CPU
    time at the same size (oracle port, 1 layer + expectation, extrapolated)."""
    import torch
    from scipy.optimize import minimize

    from paper_2309_04841_b200 import QaoaSimulator, labs_terms

    try:
        n, p = 30, 10
        t0 = time.perf_counter()
        sim = QaoaSimulator(terms=labs_terms(n))
        torch.cuda.synchronize()
        pre = time.perf_counter() - t0
        x0 = np.concatenate(angles(p)) * 0.1
        calls = [0]

        def f(x):
            calls[0] += 1
            return sim.objective(x[:p], x[p:])

        f(x0)
        torch.cuda.synchronize()
        calls[0] = 0
        t0 = time.perf_counter()
        res = minimize(f, x0, method="COBYLA", options={"maxiter": args.cobyla_iters, "rhobeg": 0.05})
        dt = time.perf_counter() - t0
        ms_dev = _event_ms(lambda: sim.objective(res.x[:p], res.x[p:]), 2, 1)
        out = {"workload": "LABS n=30 p=10 X-mixer complex128 objective inside scipy COBYLA "
                           f"(maxiter {args.cobyla_iters}, rhobeg 0.05, x0 = 0.1 * default_rng(0) U(0,1))",
               "evals": calls[0], "wall_s": dt, "evals_per_s": calls[0] / dt, "ms_per_eval_device": ms_dev,
               "precompute_s": pre, "objective_start": float(f(x0)), "objective_end": float(res.fun),
               "cost_encoding": "uint16" if sim.device_costs.u16 is not None else "float64"}
        del sim
        torch.cuda.empty_cache()
        return out
    except Exception as exc:  # noqa: BLE001 - an extra key never fails the headline line
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}


def run_config1():
    """BASELINE config 1: LABS n=12 p=4 (the reference's CPU-runnable case): device
    time of one evaluation back to back (the one-CTA resident kernel) and the
    batched throughput (4096 parameter sets, one CTA each)."""
    import torch

    from paper_2309_04841_b200 import QaoaSimulator, labs_terms

    try:
        n, p = 12, 4
        g, b = angles(p)
        sim = QaoaSimulator(terms=labs_terms(n))
        rng = np.random.default_rng(1)
        B = 4096
        G, Bt = rng.uniform(0, 1, (B, p)), rng.uniform(0, 1, (B, p))
        for _ in range(50):
            sim.simulate_qaoa_batched(G, Bt)
        ms1 = _event_ms(lambda: sim.simulate_qaoa(g, b, reuse_buffer=True), 200, 1)
        msb = _event_ms(lambda: sim.simulate_qaoa_batched(G, Bt), 10, 1)
        for _ in range(20):  # the first call at a depth captures the evaluation's CUDA graph
            sim.objective(g, b)
        t0 = time.perf_counter()
        for _ in range(500):
            sim.objective(g, b)
        call_ms = (time.perf_counter() - t0) / 500 * 1e3
        out = {"workload": "LABS n=12 p=4 X-mixer complex128", "device_us_per_eval": ms1 * 1e3,
               "objective_call_us": call_ms * 1e3, "batched_evals_per_s": B / (msb / 1e3), "batch": B}
        del sim
        torch.cuda.empty_cache()
        return out
    except Exception as exc:  # noqa: BLE001 - an extra key never fails the headline line
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}


def run_config2():
    """BASELINE config 2: MaxCut random 3-regular n=26 p=6 (the committed graph
    tests/golden/maxcut26.edges), evals/s and the HBM roofline of the step."""
    import torch

    from paper_2309_04841_b200 import Graph, QaoaSimulator, _lib, maxcut_terms
    from paper_2309_04841_b200.mixers import run_program

    try:
        with open(os.path.join(ROOT, "tests", "golden", "maxcut26.edges")) as f:
            edges = [tuple(int(x) for x in ln.split()) for ln in f if ln.strip() and not ln.startswith("#")]
        n, p = 26, 6
        g, b = angles(p)
        sim = QaoaSimulator(terms=maxcut_terms(Graph.from_edges(n, edges)))
        dc = sim.device_costs
        state = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
        e = torch.empty(1, dtype=torch.float64, device="cuda")
        layers = [(float(x), float(y), 1, 0, n) for x, y in zip(g, b)]
        fn = lambda: run_program(state, n, "x", layers, dc=dc, init=True,  # noqa: E731
                                 init_amp=1 / math.sqrt(1 << n), expectation_out=e)
        for _ in range(3):
            fn()
        ms = _event_ms(fn, 20, 1)
        lay = (_lib.FqLayer * p)(*[_lib.FqLayer(*t) for t in layers])
        passes = _lib.load().fq_plan_x_passes(n, p, lay, 0)
        S, C = 16 << n, dc.nbytes_per_amp() << n
        byts = passes * 2 * S - S + (p + 1) * C
        peak, _ = load_peaks()
        out = {"workload": "MaxCut 3-regular n=26 p=6 X-mixer complex128 objective", "ms_per_eval": ms,
               "evals_per_s": 1e3 / ms, "passes_per_eval": passes, "hbm_bytes_per_eval": byts,
               "roofline_frac_hbm": byts / (ms / 1e3) / 1e9 / peak, "objective": float(e.item()),
               "cost_encoding": "uint16" if dc.u16 is not None else "float64"}
        del sim, dc, state
        torch.cuda.empty_cache()
        return out
    except Exception as exc:  # noqa: BLE001
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}


def run_config4():
    """BASELINE config 4: portfolio n=26 (float64 costs) under the XY-ring and
    XY-complete mixers from the Hamming-weight-13 state: device ms per layer
    (p = 4 in place, phase + mixer) and the HBM roofline of the tiled XY passes."""
    import torch

    from paper_2309_04841_b200 import QaoaSimulator, _lib, hamming_weight_state
    from paper_2309_04841_b200.mixers import run_program
    from paper_2309_04841_b200.problems import portfolio_terms

    try:
        n, p = 26, 4
        g, b = angles(p)
        sim = QaoaSimulator(terms=portfolio_terms(n))
        dc = sim.device_costs
        init = torch.from_numpy(hamming_weight_state(n, n // 2)).cuda()
        peak, _ = load_peaks()
        out = {"workload": "portfolio n=26 (float64 costs), Hamming weight 13, p=4 in place"}
        for kind in ("xy-ring", "xy-complete"):
            state = init.clone()
            e = torch.empty(1, dtype=torch.float64, device="cuda")
            layers = [(float(x), float(y), 1, 0, n) for x, y in zip(g, b)]
            fn = lambda: run_program(state, n, kind, layers, dc=dc, expectation_out=e)  # noqa: E731
            fn()
            ms = _event_ms(fn, 3, 1) / p
            rounds = ctypes.c_int()
            passes = _lib.load().fq_plan_xy_passes(n, _lib.MIXER_CODES[kind], ctypes.byref(rounds))
            S, C = 16 << n, dc.nbytes_per_amp() << n
            byts = passes * 2 * S + C  # per layer: every pass reads + writes the state, the phase reads the costs
            out[kind] = {"ms_per_layer": ms, "passes_per_layer": passes, "register_rounds_per_layer": rounds.value,
                         "hbm_bytes_per_layer": byts, "roofline_frac_hbm": byts / (ms / 1e3) / 1e9 / peak}
            del state
        del sim, dc, init
        torch.cuda.empty_cache()
        return out
    except Exception as exc:  # noqa: BLE001
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}


def run_config5(args, world, rank, k, barrier):
    """BASELINE config 5 / north star: LABS n=34 p=10 complex128 sharded over the
    N ranks (fused sharded program: local passes on each shard, global-group
    passes spanning all shards over NVLink).  Per-layer ms and HBM roofline per
    GPU (algorithmic bytes of the rank's passes / time).  One GPU cannot hold
    the complex128 state (256 GiB): N = 1 reports complex64 n=34 (128 GiB), the
    same problem at the optional precision.  The reference refuses n > 30
    (terms.py:23), so there is no CPU point at this size."""
    import torch

    from paper_2309_04841_b200 import QaoaSimulator, _lib, labs_terms
    from paper_2309_04841_b200.distributed import ShardedQaoaSimulator

    n, p = 34, 10
    g, b = angles(p)
    try:
        free, _ = torch.cuda.mem_get_info()
        if os.environ.get("FQ_BENCH_ONE_DEVICE") == "1":
            free //= world  # validation mode: every rank shares one device
        c64 = world == 1
        elem = 8 if c64 else 16
        n_local = n - k
        fits = (1 << n_local) * (elem + 2) <= 0.92 * free
        if world > 1:  # every rank takes the same branch (the constructor below is collective)
            import torch.distributed as dist

            flag = torch.tensor([1 if fits else 0], dtype=torch.int32, device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            fits = bool(flag.item())
        if not fits:
            return {"skipped": f"n=34 needs {(1 << n_local) * (elem + 2) / 2**30:.0f} GiB per GPU, "
                               f"{free / 2**30:.0f} GiB free on this rank"}
        t0 = time.perf_counter()
        if world == 1:
            sim = QaoaSimulator(terms=labs_terms(n), dtype="complex64")
            fn = lambda: sim.objective(g, b)  # noqa: E731
        else:
            sim = ShardedQaoaSimulator(labs_terms(n), global_mode="fused")
            fn = lambda: sim.simulate_qaoa(g, b)  # noqa: E731
        barrier()
        pre = time.perf_counter() - t0
        obj = float(fn())
        ms = _event_ms(fn, 1, world)
        S = elem * (1 << n_local)
        lay = (_lib.FqLayer * p)(*[_lib.FqLayer(float(gi), float(bi), 1, 0, n) for gi, bi in zip(g, b)])
        gp = ctypes.c_int()
        if world == 1:
            passes = _lib.load().fq_plan_x_passes(n, p, lay, _lib.STATE_C64)
            gpv = 0
        else:
            passes = _lib.load().fq_plan_sharded_passes(n_local, k, p, lay, ctypes.byref(gp))
            gpv = gp.value
        C = 2 * (1 << n_local)
        hbm = passes * 2 * S - S + (p + 1) * C
        peak, _ = load_peaks()
        out = {"workload": f"LABS n=34 p=10 X-mixer {'complex64 (complex128 needs 256 GiB)' if c64 else 'complex128'}"
                           f" on {world} GPU(s), n_local={n_local}",
               "ms_per_eval": ms, "ms_per_layer": ms / p, "precompute_s": pre, "objective": obj,
               "passes_per_eval": passes, "spanning_passes_per_eval": gpv,
               "hbm_bytes_per_gpu": hbm, "nvlink_bytes_per_gpu": gpv * 2 * S * (world - 1) // world,
               "roofline_frac_hbm": hbm / (ms / 1e3) / 1e9 / peak,
               "cpu_reference": "n/a: the reference refuses n > 30 (terms.py:23, MemoryError)"}
        del sim
        torch.cuda.empty_cache()
        return out
    except Exception as exc:  # noqa: BLE001 - an extra key never fails the headline line
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}


# ---------------------------------------------------------------------------- GPU
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--qubits", "--n", dest="n", type=int, default=0, help="total qubits (default 26 + log2 N)")
    ap.add_argument("--p", type=int, default=10)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--global-mode", default="fused", choices=["fused", "p2p", "exchange"],
                    help="N>1: one sharded program whose global-qubit passes span all shards over peer memory "
                         "(fused), a per-layer peer-memory global kernel (p2p), or NCCL all-to-all exchanges")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the extra BASELINE config keys (config3: COBYLA loop at n=30; config5: LABS n=34)")
    ap.add_argument("--cobyla-iters", type=int, default=24)
    ap.add_argument("--state", default="c128", choices=["c128", "c64"],
                    help="state type: complex128 (the headline, the reference's) or the optional complex64")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    # FQ_BENCH_ONE_DEVICE=1: validation of the multi-process path on a one-GPU box
    # (every rank on cuda:0, gloo for the host-side collectives; timings not meaningful)
    one_device = os.environ.get("FQ_BENCH_ONE_DEVICE") == "1"
    if one_device:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_device:
            dist.init_process_group("gloo")
        else:
            # NCCL's communicator lines (nRanks, NVLink / NVLS transports) on stderr: the
            # evidence that N ranks really formed one communicator over this node's GPUs
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2309_04841_b200 import QaoaSimulator, _lib, labs_terms
    from paper_2309_04841_b200.distributed import ShardedQaoaSimulator
    from paper_2309_04841_b200.mixers import run_program

    k = int(math.log2(world))
    n = args.n or (BASE_N + k)
    p = args.p
    g, b = angles(p)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ------------------------------------------------------------ setup (+ precompute, timed separately)
    barrier()
    t0 = time.perf_counter()
    poly = labs_terms(n)
    c64 = args.state == "c64"
    if c64 and world > 1 and args.global_mode != "fused":
        raise SystemExit("--state c64 on several GPUs needs --global-mode fused")
    if world == 1:
        sim = QaoaSimulator(terms=poly, dtype=torch.complex64 if c64 else torch.complex128)
        dc = sim.device_costs
    else:
        sim = ShardedQaoaSimulator(poly, global_mode=args.global_mode,
                                   dtype=torch.complex64 if c64 else torch.complex128)
        if args.global_mode == "fused" and not c64:
            # the fused mode maps every rank's shard over CUDA IPC; if that is not
            # possible on this node, all ranks fall back to NCCL exchanges together
            ok = 1
            try:
                sim.simulate_qaoa(g, b, expectation=False)
                torch.cuda.synchronize()
                sim.check_barrier()
            except Exception as exc:  # noqa: BLE001 - reported, then the exchange path runs
                print(f"[bench] rank {rank}: fused sharded mode failed ({type(exc).__name__}: {exc}); "
                      f"falling back to global_mode='exchange'", file=sys.stderr, flush=True)
                ok = 0
            flag = torch.tensor([ok], dtype=torch.int32, device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 0:
                args.global_mode = "exchange"
                args.fallback = True
                sim = ShardedQaoaSimulator(poly, global_mode="exchange")
        dc = sim.costs
    barrier()
    precompute_s = time.perf_counter() - t0
    n_local = n - k
    S = (8 if c64 else 16) * (1 << n_local)
    Cb = dc.nbytes_per_amp() * (1 << n_local)

    # ------------------------------------------------------------ device-resident step
    layers = [(float(gi), float(bi), 1, 0, n_local) for gi, bi in zip(g, b)]
    if world == 1:
        state = torch.empty(1 << n, dtype=torch.complex64 if c64 else torch.complex128, device="cuda")
        exp_dev = torch.empty(1, dtype=torch.float64, device="cuda")
        amp = 1.0 / math.sqrt(float(1 << n))

        def step():
            run_program(state, n, "x", layers, dc=dc, init=True, init_amp=amp, expectation_out=exp_dev)
    else:
        def step():
            # the public call: one sharded program whose last pass accumulates this rank's
            # objective partials, then one all-reduce (objective + barrier error word)
            sim.simulate_qaoa(g, b)

    for _ in range(args.warmup):
        step()
    barrier()
    # e2e through the public API (one GPU): fresh host angles every step, the scalar read back
    e2e_ms = None
    if world == 1:
        rng_e = np.random.default_rng(1)
        e2e_sets = [(g + 1e-3 * rng_e.standard_normal(p), b + 1e-3 * rng_e.standard_normal(p))
                    for _ in range(args.steps + args.warmup)]

        def e2e_step(i):
            res = sim.simulate_qaoa(*e2e_sets[i])
            val = sim.get_expectation(res)
            del res
            return val
    # the device-resident steps and the e2e steps run interleaved in blocks when two
    # states fit (the pool's boxes drift with power capping over a run: measuring one
    # arm after the other would bias the later one)
    interleave = world == 1 and 2 * S_total_bytes(n, c64) < 0.8 * torch.cuda.mem_get_info()[0]
    if interleave:
        for i in range(args.warmup):
            e2e_step(i)
        barrier()
    blocks = [args.steps // 4 + (1 if i < args.steps % 4 else 0) for i in range(4)] if interleave else [args.steps]
    blocks = [x for x in blocks if x > 0]
    sampler = ClockSampler(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = 0.0
    e2e_ms_sum = 0.0
    e2e_i = args.warmup
    with sampler:
        for blk in blocks:
            e0.record(stream)
            for _ in range(blk):
                step()
            e1.record(stream)
            barrier()
            ms += e0.elapsed_time(e1)
            if interleave:
                t_wall = time.perf_counter()
                e0.record(stream)
                for _ in range(blk):
                    e2e_step(e2e_i)
                    e2e_i += 1
                e1.record(stream)
                torch.cuda.synchronize()
                e2e_ms_sum += max(e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t_wall))
    if interleave:
        e2e_ms = e2e_ms_sum
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    # unit of work: weak scaling (default, n = 26 + log2 N) counts n=26-equivalent evaluations,
    # so ideal scaling is N x the 1-GPU value; a fixed --qubits problem counts evaluations of it
    # at every N (strong scaling) — the same unit at every world size
    units_per_eval = 1.0 if args.n else 2.0 ** (n - BASE_N)
    value = args.steps * units_per_eval / (ms / 1e3)

    # ------------------------------------------------------------ byte model of the step (per GPU)
    lay = (_lib.FqLayer * p)(*[_lib.FqLayer(*lt) for lt in layers])
    skind = _lib.STATE_C64 if c64 else _lib.STATE_C128
    passes = _lib.load().fq_plan_x_passes(n_local, p, lay, skind)
    n_phase = sum(1 for gi in g if gi != 0.0)
    P_survey = -(-n_local // 12)
    survey_bytes = p * (P_survey * 2 * S + Cb) + (S + Cb)
    if world == 1:
        # HBM round trips of the state actually run: the planned passes, minus one per
        # L2 slab sweep (a sweep runs two passes over each L2-resident slab)
        step()
        torch.cuda.synchronize()
        round_trips = _lib.load().fq_last_passes(None, None, 0)
        sweeps = passes - round_trips
        tile_bytes = round_trips * 2 * S - S + (n_phase + 1) * Cb  # first pass generates |+>, last reads costs for E
        launches = round_trips + 1 + sweeps  # + the partials' sum, + one counter memset per sweep
    elif args.global_mode == "fused":
        # one sharded plan over all n qubits; its global-group passes span the shards
        glay = (_lib.FqLayer * p)(*[_lib.FqLayer(float(gi), float(bi), 1, 0, n) for gi, bi in zip(g, b)])
        gp = ctypes.c_int()
        passes = _lib.load().fq_plan_sharded_passes(n_local, k, p, glay, ctypes.byref(gp))
        tile_bytes = passes * 2 * S - S + (n_phase + 1) * Cb  # the last pass reads the costs for E (fused)
        launches = passes + 2 * gp.value + 1  # + two device barriers per spanning pass, + the partials' sum
        nvlink_bytes = gp.value * 2 * S * (world - 1) // world
    else:
        post = p * (1 if k > 0 else 0)  # the k-position pass after each exchange
        per_layer = _lib.load().fq_plan_x_passes(n_local, 1, lay, skind)
        tile_bytes = p * per_layer * 2 * S - S + n_phase * Cb + post * 2 * S + S + Cb
        launches = p * (per_layer + (1 if k > 0 else 0)) + 2
    peak, peak_kind = load_peaks()
    achieved_step = tile_bytes / (ms_step / 1e3) / 1e9

    # ------------------------------------------------------------ per-launch timing of the pass kernel
    # CUDA events recorded by libfqaoa between consecutive passes on the launching
    # stream (option "time_passes"), over `steps` extra steps right after the
    # timed region; achieved = algorithmic bytes of the passes / their event time.
    kinds = {}
    if world == 1:
        _lib.call("fq_set_option", b"time_passes", 1)
        info = (ctypes.c_int * (5 * 256))()
        tms = (ctypes.c_float * 256)()
        tot_b = tot_ms = 0.0
        for _ in range(args.steps):
            step()
            cnt = _lib.load().fq_last_passes(info, tms, 256)
            for i in range(cnt):
                sq, ph, nt, ini, ex = info[5 * i:5 * i + 5]
                nb = (0 if ini else S) + S + (Cb if (ph or ex) else 0)
                kd = kinds.setdefault(pass_name(sq) + (" +phase" if ph in (1, 2) else "") +
                                      (" +init" if ini else "") + (" +expect" if ex else ""),
                                      {"launches": 0, "ms": 0.0, "bytes": 0})
                kd["launches"] += 1
                kd["ms"] += tms[i]
                kd["bytes"] += nb
                tot_b += nb
                tot_ms += tms[i]
        _lib.call("fq_set_option", b"time_passes", 0)
        for kd in kinds.values():
            kd["avg_ms"] = kd["ms"] / kd["launches"]
            kd["GBps"] = kd["bytes"] / (kd["ms"] / 1e3) / 1e9
            kd["bytes_per_launch"] = kd["bytes"] // kd["launches"]
            del kd["ms"], kd["bytes"]
        achieved = tot_b / (tot_ms / 1e3) / 1e9 if tot_ms > 0 else achieved_step
    else:
        achieved = achieved_step

    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                tj = json.load(f)
            if tj.get("n") == n_local and tj.get("state", "c128") == args.state:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ------------------------------------------------------------ e2e through the public API
    e2e = None
    if world == 1:
        objective = float(exp_dev.item())
        del step, state  # the API allocates its own state (n = 34 complex64: no room for two)
        if e2e_ms is None:  # not interleaved (two states do not fit): the e2e arm after the device arm
            for i in range(args.warmup):
                e2e_step(i)
            barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t_wall = time.perf_counter()
            f0.record(stream)
            for i in range(args.warmup, args.warmup + args.steps):
                e2e_step(i)
            f1.record(stream)
            torch.cuda.synchronize()
            t_wall = time.perf_counter() - t_wall
            e2e_ms = max(f0.elapsed_time(f1), 1e3 * t_wall)
        e2e = {"value": args.steps / (e2e_ms / 1e3), "unit": "evals/s", "h2d_bytes_per_step": 2 * p * 8,
               "d2h_bytes_per_step": 8, "ms_per_step": e2e_ms / args.steps,
               "api": "QaoaSimulator.simulate_qaoa + get_expectation",
               "timing": ("interleaved with the device-resident steps in 4 blocks" if interleave
                          else "after the device-resident steps")}
    else:
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            sim.simulate_qaoa(g, b, expectation=True)
        f1.record(stream)
        barrier()
        t = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        e2e = {"value": args.steps * units_per_eval / (e2e_ms / 1e3), "unit": "evals/s",
               "h2d_bytes_per_step": 2 * p * 8, "d2h_bytes_per_step": 8, "ms_per_step": e2e_ms / args.steps,
               "api": "ShardedQaoaSimulator.simulate_qaoa"}

    # ------------------------------------------------------------ N > 1: fused vs NCCL exchange, same run
    crosscheck = None
    if world > 1:
        objective_fused = float(sim.simulate_qaoa(g, b))
        if args.global_mode == "fused" and not c64:
            try:
                xsim = ShardedQaoaSimulator(poly, global_mode="exchange")
                obj_x = float(xsim.simulate_qaoa(g, b))
                crosscheck = {"fused_objective": objective_fused, "nccl_exchange_objective": obj_x,
                              "rel_diff": abs(objective_fused - obj_x) / max(1e-300, abs(obj_x)),
                              "exchanges_per_eval": xsim.exchange_count}
                del xsim
            except Exception as exc:  # noqa: BLE001 - reported in the line
                crosscheck = {"error": f"{type(exc).__name__}: {exc}"[:300]}
            torch.cuda.empty_cache()

    # ------------------------------------------------------------ CPU baseline (rank 0, N = 1 only)
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu:
        from oracle import oracle as O

        costs_host = sim.get_cost_diagonal()
        layers_sample = 2
        rate, t_layer, t_exp = cpu_eval_rate(np.array(costs_host), p, g, b, layers_sample)
        cpu = {"value": rate, "unit": "evals/s", "cores": O.num_threads(), "kind": "port", "cpu": cpu_model(),
               "sample": f"{layers_sample} of {p} layers (phase + X mixer) + 1 expectation of LABS n={n} on the "
                         f"oracle C/OpenMP port, extrapolated to the p={p} evaluation "
                         f"({1e3 * t_layer:.0f} ms/layer, {1e3 * t_exp:.0f} ms expectation)"}

    if world > 1:
        objective = float(sim.expectation())  # collective

    # ------------------------------------------------------------ BASELINE configs 3 and 5 (extra keys)
    cost_encoding = "uint16 levels (lossless)" if dc.u16 is not None else "float64"
    extra = {}
    if not args.no_configs:
        del sim, dc
        torch.cuda.empty_cache()
        if world == 1:
            extra["config1"] = run_config1()
            extra["config2"] = run_config2()
            extra["config3"] = run_config3(args)
            extra["config4"] = run_config4()
        extra["config5"] = run_config5(args, world, rank, k, barrier)
    if rank == 0:
        line = {
            **({"validation_only": "all ranks on one GPU (FQ_BENCH_ONE_DEVICE)"} if one_device else {}),
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if args.n else "weak",  # --qubits fixes the total problem
            "vs_baseline": None, "dtype": args.state, "data": "synthetic",
            "config": {"workload": f"LABS n={n} p={p} X-mixer {'complex64' if c64 else 'complex128'} objective evaluation"
                                   + (f" sharded over {world} GPUs (n_local={n_local}; value in n=26-equivalent "
                                      f"evaluations)" if world > 1 else ""),
                       "n": n, "p": p, "n_local": n_local, "angles": "default_rng(0) U(0,1)",
                       "cost_encoding": cost_encoding,
                       "l2": (f"no flush: {S / 2**30:.2f} GiB state per GPU >> 126 MB L2" if S > (256 << 20)
                              else f"state of {S >> 20} MiB per GPU is L2-sized (validation sizes only)"),
                       "parallelism": (f"state sharded over {world} GPUs by global qubits, global-qubit mixer: "
                                       + {"fused": "passes spanning all shards over peer memory (CUDA IPC, NVLink), "
                                                   "fused across layers",
                                          "p2p": "per-layer peer-memory kernel (CUDA IPC over NVLink)",
                                          "exchange": "NCCL all-to-all"}[args.global_mode])
                                      if world > 1 else "single GPU",
                       **({"nvlink_bytes_per_step": nvlink_bytes, "spanning_passes_per_step": gp.value}
                          if world > 1 and args.global_mode == "fused" else {}),
                       **({"fallback": "fused mode failed on this node; NCCL exchange path measured"}
                          if getattr(args, "fallback", False) else {})},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                         "kernel": "k_pass16 (every tiled pass of the step; per-launch CUDA events)",
                         "bytes_per_launch": f"2*S + C(phase/expectation) - S(|+> generated); S = {S >> n_local}*2^n, "
                                             "C = cost bytes per amplitude * 2^n",
                         "achieved_whole_step": achieved_step,
                         "algorithmic_bytes_per_step": tile_bytes, "passes_per_step": passes if world == 1 else None,
                         **({"hbm_round_trips_per_step": round_trips, "l2_sweeps_per_step": sweeps,
                             "l2_note": "a sweep runs two passes per L2-resident slab: its second pass reads and "
                                        "writes L2, not HBM (algorithmic HBM bytes count one round trip)"}
                            if world == 1 else {}),
                         "by_pass_kind": kinds or None,
                         "survey_model": {"bytes_per_eval": survey_bytes, "evals_per_s_at_peak": peak * 1e9 / survey_bytes,
                                          "note": "SURVEY.md §8(d): P=ceil(n/12) unfused passes per layer"}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches * args.steps,
            "clocks": sampler.summary(),
            **({"crosscheck": crosscheck} if crosscheck else {}),
            **extra,
            "precompute_s": precompute_s,
            "ms_per_layer": ms_step / p,
            "objective": objective,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
