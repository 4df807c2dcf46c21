"""Randomised multi-process stress run of ShardedQaoaSimulator(global_mode="fused")
(development tool): 2 or 4 ranks on the visible GPU(s) (all on cuda:0 when only
one is visible; gloo carries the host collectives), random n, depth, mixer and
state type, each compared with the single-GPU simulator.  Exits 1 on failure."""

import os
import socket
import sys
import time

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup(seed):
    from paper_2309_04841_b200.mixers import SU2, Mixer
    from paper_2309_04841_b200.problems import labs_terms, portfolio_terms

    rng = np.random.default_rng(seed)
    world = [2, 4][int(rng.integers(0, 2))]
    k = world.bit_length() - 1
    n = int(rng.integers(12 + k, 19))
    p = int(rng.integers(1, 4))
    kind = ["x", "custom", "xy-ring", "xy-complete"][int(rng.integers(0, 4))]
    dtype = "complex64" if (kind != "custom" and rng.random() < 0.3) else None
    g, b = rng.uniform(-1, 1, p), rng.uniform(-1.5, 1.5, p)
    poly = portfolio_terms(n) if kind.startswith("xy") or rng.random() < 0.3 else labs_terms(n)
    mix = Mixer.custom(lambda beta: [SU2(np.cos(beta * (1 + 0.07 * j)), -1j * np.sin(beta * (1 + 0.07 * j)))
                                     for j in range(n)]) if kind == "custom" else Mixer(kind)
    w = n // 2 if kind.startswith("xy") else None
    return world, n, p, kind, dtype, g, b, poly, mix, w


def _worker(rank, world, port, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_04841_b200.distributed import ShardedQaoaSimulator

        _, n, p, kind, dtype, g, b, poly, mix, w = _setup(seed)
        sim = ShardedQaoaSimulator(poly, mixer=mix, global_mode="fused", dtype=dtype)
        E = sim.simulate_qaoa(g, b, initial_weight=w)
        q.put((rank, E, sim.shard.cpu().numpy()))
        dist.barrier()
        sim.close()
    except Exception as exc:  # noqa: BLE001
        q.put((rank, None, repr(exc)))
    finally:
        dist.destroy_process_group()


def one(seed):
    from paper_2309_04841_b200 import QaoaSimulator, hamming_weight_state

    world, n, p, kind, dtype, g, b, poly, mix, w = _setup(seed)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
    if any(o[1] is None for o in out):
        return False, {"errors": [o[2] for o in out if o[1] is None], "world": world, "n": n, "kind": kind}
    sim = QaoaSimulator(terms=poly, mixer=mix)
    init = hamming_weight_state(n, w) if w is not None else None
    res = sim.simulate_qaoa(g, b, initial=init)
    full = np.concatenate([o[2] for o in out]).astype(np.complex128)
    tol = 1e-4 * np.abs(res.state).max() if dtype else 1e-12
    err = np.abs(full - res.state).max()
    e_ref = sim.get_expectation(res)
    dE = max(abs(o[1] - e_ref) for o in out)
    ok = err <= tol and dE <= (1e-4 * max(1.0, abs(e_ref)) if dtype else 1e-10 * max(1.0, abs(e_ref)))
    return ok, {"world": world, "n": n, "p": p, "kind": kind, "dtype": dtype, "err": err, "dE": dE}


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    t0, seed, runs, fails = time.time(), 500, 0, 0
    while time.time() - t0 < budget:
        seed += 1
        ok, info = one(seed)
        runs += 1
        if not ok:
            fails += 1
            print("FAIL seed", seed, info, flush=True)
    print(f"stress_mp: {runs} random sharded programs, {fails} failures, {time.time() - t0:.0f} s", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
