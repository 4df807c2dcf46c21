"""Kernel-variant timing harness (development tool, not the driver bench).

Times the fused LABS program at n (default 26) under each option combination
and prints ms/step, ms/pass and effective GB/s of the pass stream."""

import argparse
import ctypes
import itertools
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_04841_b200 import QaoaSimulator, _lib, labs_terms  # noqa: E402
from paper_2309_04841_b200.mixers import run_program  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=26)
    ap.add_argument("--p", type=int, default=10)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--opts", default="plan=0,1")
    ap.add_argument("--detail", action="store_true", help="per-pass CUDA-event times of one step")
    ap.add_argument("--state", default="c128", choices=["c128", "c64"])
    args = ap.parse_args()
    n, p = args.n, args.p
    dt = torch.complex64 if args.state == "c64" else torch.complex128
    sim = QaoaSimulator(terms=labs_terms(n), dtype=dt)
    dc = sim.device_costs
    rng = np.random.default_rng(0)
    g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
    state = torch.empty(1 << n, dtype=dt, device="cuda")
    e = torch.empty(1, dtype=torch.float64, device="cuda")
    S = (8 if args.state == "c64" else 16) * (1 << n)
    C = dc.nbytes_per_amp() * (1 << n)
    opts = [o.split("=") for o in args.opts.split(";") if o]
    names = [o[0] for o in opts]
    for combo in itertools.product(*[o[1].split(",") for o in opts]):
        for nm, v in zip(names, combo):
            _lib.call("fq_set_option", nm.encode(), int(v))
        for label, gam in (("phase", g), ("nophase", np.zeros(p))):
            layers = [(float(x), float(y), 1, 0, n) for x, y in zip(gam, b)]
            lay = (_lib.FqLayer * p)(*[_lib.FqLayer(*t) for t in layers])
            passes = _lib.load().fq_plan_x_passes(n, p, lay, _lib.STATE_C64 if args.state == "c64" else 0)
            if args.detail or True:  # HBM round trips actually run (sweeps fuse pass pairs)
                fn0 = lambda: run_program(state, n, "x", layers, dc=dc, init=True, init_amp=1 / math.sqrt(1 << n),
                                          expectation_out=e)
                fn0()
                passes = _lib.load().fq_last_passes(None, None, 0)
            fn = lambda: run_program(state, n, "x", layers, dc=dc, init=True, init_amp=1 / math.sqrt(1 << n),
                                     expectation_out=e)
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(args.steps):
                fn()
            t1.record()
            torch.cuda.synchronize()
            ms = t0.elapsed_time(t1) / args.steps
            nph = int(np.count_nonzero(gam))
            byts = passes * 2 * S - S + (nph + 1) * C
            print(json.dumps({"opts": dict(zip(names, combo)), "mode": label, "ms_step": round(ms, 3),
                              "passes": passes, "ms_pass": round(ms / passes, 4),
                              "GBps": round(byts / ms / 1e6, 1), "E": float(e.item())}), flush=True)
            if args.detail:
                _lib.call("fq_set_option", b"time_passes", 1)
                fn()
                info = (ctypes.c_int * (5 * 64))()
                tms = (ctypes.c_float * 64)()
                cnt = _lib.load().fq_last_passes(info, tms, 64)
                _lib.call("fq_set_option", b"time_passes", 0)
                names_seq = {-1: "phase", 0: "8|0|4", 1: "8|4", 2: "8|0|4|0|8", 3: "8|4|8"}
                for a in range(4):
                    for c in range(4):
                        names_seq[100 + 10 * a + c] = f"[{names_seq[a]}>{names_seq[c]}]"
                for i in range(cnt):
                    sq, ph, nt, ini, ex = info[5 * i:5 * i + 5]
                    nb = (0 if ini else S) + S + (C if (ph or ex) else 0)
                    print(f"    pass {i:2d} {names_seq[sq]:10s} ph={ph} targets={nt:2d} init={ini} exp={ex} "
                          f"{tms[i]:.4f} ms {nb / tms[i] / 1e6:7.1f} GB/s", flush=True)
    for nm in names:
        _lib.call("fq_set_option", nm.encode(), 1)


if __name__ == "__main__":
    main()
