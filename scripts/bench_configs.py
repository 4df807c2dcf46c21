"""BASELINE.json configurations beyond the headline (bench.py), single B200,
each next to the CPU oracle port on this host's cores (bounded samples).
One JSON line per configuration.

    python scripts/bench_configs.py [--only 1,2,3,4,5] [--skip-cpu]

1. LABS n=12 p=4 X mixer — latency of one evaluation and the batched
   (one CTA per parameter set) throughput for optimiser sweeps.
2. MaxCut random 3-regular n=26 p=6 (pinned edge list, tests/golden/maxcut26.edges).
3. LABS n=30 p=10 inside a COBYLA loop (scipy.optimize.minimize), precompute
   once; evals/s including the host round trip of every evaluation.
4. Portfolio n=26, XY-ring and XY-complete mixers, Hamming-weight-13 start.
5. Capacity anchor for the sharded n=34 run: LABS n=33 p=10 on ONE B200
   (uint16 diagonal, 128 GiB state; the reference refuses n > 30).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2309_04841_b200 import Mixer, QaoaSimulator, hamming_weight_state, labs_terms, maxcut_terms  # noqa: E402
from paper_2309_04841_b200.problems import Graph, portfolio_terms  # noqa: E402


def angles(p, seed=0):
    rng = np.random.default_rng(seed)
    return rng.uniform(0, 1, p), rng.uniform(0, 1, p)


def gpu_time(fn, reps, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return max(e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0)) / reps  # ms, host-inclusive


def cpu_eval(costs, g, b, kind="x", initial=None, layers_sample=None):
    """Oracle port: time `layers_sample` layers (+ one expectation), extrapolate to p."""
    from oracle import oracle as O

    n = costs.size.bit_length() - 1
    p = len(g)
    st = O.uniform_state(n) if initial is None else np.array(initial, dtype=np.complex128)
    k = p if layers_sample is None else min(p, layers_sample)
    t0 = time.perf_counter()
    for li in range(k):
        O.apply_phase(st, costs, float(g[li]))
        O.mixer_layer(st, kind, float(b[li]))
    t_layer = (time.perf_counter() - t0) / k
    t0 = time.perf_counter()
    O.expectation_fast(st, costs)
    t_exp = time.perf_counter() - t0
    return p * t_layer + t_exp, t_layer, O.num_threads()


def out(line):
    print(json.dumps(line), flush=True)


def config1(args):
    n, p = 12, 4
    g, b = angles(p)
    sim = QaoaSimulator(terms=labs_terms(n))
    ms = gpu_time(lambda: sim.get_expectation(sim.simulate_qaoa(g, b)), 200)
    B = 4096
    rng = np.random.default_rng(1)
    G, Bt = rng.uniform(0, 1, (B, p)), rng.uniform(0, 1, (B, p))
    ms_b = gpu_time(lambda: sim.simulate_qaoa_batched(G, Bt), 5)
    line = {"config": "1: LABS n=12 p=4 X", "gpu_latency_ms": ms, "gpu_evals_per_s_single": 1e3 / ms,
            "gpu_evals_per_s_batched": B / (ms_b / 1e3), "batch": B}
    if not args.skip_cpu:
        t, _, cores = cpu_eval(sim.get_cost_diagonal(), g, b)
        reps = max(1, int(0.5 / t))
        t0 = time.perf_counter()
        for _ in range(reps):
            cpu_eval(sim.get_cost_diagonal(), g, b)
        t = (time.perf_counter() - t0) / reps
        line.update({"cpu_evals_per_s": 1 / t, "cpu_cores": cores, "cpu_kind": "oracle port (C/OpenMP)"})
    out(line)


def config2(args):
    with open(os.path.join(ROOT, "tests", "golden", "maxcut26.edges")) as f:
        edges = [tuple(int(x) for x in ln.split()) for ln in f if ln.strip() and not ln.startswith("#")]
    n, p = 26, 6
    g, b = angles(p)
    t0 = time.perf_counter()
    sim = QaoaSimulator(terms=maxcut_terms(Graph.from_edges(n, edges)))
    torch.cuda.synchronize()
    pre = time.perf_counter() - t0
    ms = gpu_time(lambda: sim.get_expectation(sim.simulate_qaoa(g, b, reuse_buffer=True)), 20)
    line = {"config": "2: MaxCut 3-regular n=26 p=6 X", "gpu_ms_per_eval": ms, "gpu_evals_per_s": 1e3 / ms,
            "precompute_s": pre, "cost_encoding": "uint16" if sim.device_costs.u16 is not None else "float64"}
    if not args.skip_cpu:
        t, tl, cores = cpu_eval(sim.get_cost_diagonal(), g, b, layers_sample=1)
        line.update({"cpu_evals_per_s": 1 / t, "cpu_cores": cores, "cpu_sample": "1 layer + expectation, extrapolated"})
    out(line)


def config3(args):
    from scipy.optimize import minimize

    n, p = 30, 10
    t0 = time.perf_counter()
    sim = QaoaSimulator(terms=labs_terms(n))
    torch.cuda.synchronize()
    pre = time.perf_counter() - t0
    x0 = np.concatenate(angles(p)) * 0.1
    calls = []

    def f(x):
        calls.append(1)
        return sim.get_expectation(sim.simulate_qaoa(x[:p], x[p:], reuse_buffer=True))

    f(x0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = minimize(f, x0, method="COBYLA", options={"maxiter": args.cobyla_iters, "rhobeg": 0.05})
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    line = {"config": "3: LABS n=30 p=10 in COBYLA loop", "gpu_evals": len(calls) - 1, "gpu_wall_s": dt,
            "gpu_evals_per_s": (len(calls) - 1) / dt, "precompute_s": pre, "objective_start": float(f(x0)),
            "objective_end": float(res.fun), "cost_encoding": "uint16" if sim.device_costs.u16 is not None else "float64"}
    if not args.skip_cpu:
        del sim
        from oracle import oracle as O

        # one layer of the reference algorithm at n = 30 on the host (16 GiB state)
        costs = np.zeros(1 << n)  # the layer's cost is independent of the diagonal values
        st = O.uniform_state(n)
        t0 = time.perf_counter()
        O.apply_phase(st, costs, 0.1)
        O.rx_layer(st, 0.2)
        tl = time.perf_counter() - t0
        t0 = time.perf_counter()
        O.expectation_fast(st, costs)
        te = time.perf_counter() - t0
        line.update({"cpu_evals_per_s": 1 / (p * tl + te), "cpu_cores": O.num_threads(),
                     "cpu_sample": "1 layer + expectation at n=30, extrapolated to p=10 (precompute excluded)"})
        del st, costs
    out(line)


def config4(args):
    n, p = 26, 1
    g, b = angles(p)
    poly = portfolio_terms(n)
    init = hamming_weight_state(n, n // 2)
    for kind in ("xy-ring", "xy-complete"):
        sim = QaoaSimulator(terms=poly, mixer=Mixer(kind))
        init_d = torch.from_numpy(init).cuda()
        ms = gpu_time(lambda: sim.get_expectation(sim.simulate_qaoa(g, b, initial=init_d)), 3, warm=1)
        line = {"config": f"4: portfolio n=26 {kind} p={p}", "gpu_ms_per_layer": ms, "gpu_layers_per_s": 1e3 / ms,
                "cost_encoding": "uint16" if sim.device_costs.u16 is not None else "float64"}
        # the optional complex64 state on the same problem (same diagonal)
        sim64 = QaoaSimulator(costs=sim.device_costs, mixer=Mixer(kind), dtype="complex64")
        init64 = init_d.to(torch.complex64)
        line["gpu_ms_per_layer_complex64"] = gpu_time(
            lambda: sim64.get_expectation(sim64.simulate_qaoa(g, b, initial=init64)), 3, warm=1)
        del sim64
        if not args.skip_cpu:
            from oracle import oracle as O

            costs = sim.get_cost_diagonal()
            st = np.array(init)
            edges = O.ring_edges(n) if kind == "xy-ring" else O.complete_edges(n)
            k = min(len(edges), 8)
            t0 = time.perf_counter()
            for (i, j) in edges[:k]:
                O.apply_xy(st, 0.3, i, j)
            t_gate = (time.perf_counter() - t0) / k
            t0 = time.perf_counter()
            O.apply_phase(st, costs, 0.1)
            t_ph = time.perf_counter() - t0
            t = t_ph + len(edges) * t_gate
            line.update({"cpu_ms_per_layer": 1e3 * t, "cpu_cores": O.num_threads(),
                         "cpu_sample": f"{k} of {len(edges)} gates + phase, extrapolated"})
        out(line)
        del sim


def config5(args):
    n, p = 33, 10
    g, b = angles(p)
    free, total = torch.cuda.mem_get_info()
    if (18 << n) > 0.95 * free:
        out({"config": "5: LABS n=33 p=10 on one B200", "skipped": f"needs {18 * 2**n / 2**30:.0f} GiB, "
                                                                  f"{free / 2**30:.0f} GiB free"})
        return
    t0 = time.perf_counter()
    sim = QaoaSimulator(terms=labs_terms(n))
    torch.cuda.synchronize()
    pre = time.perf_counter() - t0
    ms = gpu_time(lambda: sim.get_expectation(sim.simulate_qaoa(g, b, reuse_buffer=True)), 2, warm=1)
    S = 16 * 2 ** n
    out({"config": "5: LABS n=33 p=10 X on ONE B200 (capacity anchor; reference refuses n>30)",
         "gpu_s_per_eval": ms / 1e3, "gpu_ms_per_layer": ms / p, "precompute_s": pre,
         "state_GiB": S / 2**30, "cost_encoding": "uint16 only" if sim.device_costs.f64 is None else "f64+u16",
         "objective": float(sim.get_expectation(sim.simulate_qaoa(g, b, reuse_buffer=True)))})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="1,2,3,4,5")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--cobyla-iters", type=int, default=60)
    args = ap.parse_args()
    only = args.only.split(",")
    if len(only) > 1:  # one process per configuration: each starts with the whole device free
        import subprocess

        for c in only:
            cmd = [sys.executable, os.path.abspath(__file__), "--only", c, "--cobyla-iters", str(args.cobyla_iters)]
            subprocess.run(cmd + (["--skip-cpu"] if args.skip_cpu else []), check=False)
        return
    torch.cuda.set_device(0)
    from paper_2309_04841_b200 import _lib

    for kv in filter(None, os.environ.get("FQ_OPTS", "").split(",")):  # e.g. FQ_OPTS=xy_min_run=5
        k, v = kv.split("=")
        _lib.call("fq_set_option", k.encode(), int(v))
    fns = {"1": config1, "2": config2, "3": config3, "4": config4, "5": config5}
    try:
        fns[only[0]](args)
    except Exception as exc:
        out({"config": only[0], "error": f"{type(exc).__name__}: {exc}"})


if __name__ == "__main__":
    main()
