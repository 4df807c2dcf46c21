"""ShardedQaoaSimulator with the real CUDA shard-local path (libfqaoa) in two
processes on one B200 (the round's boxes have one GPU): gloo carries the
exchange through host memory, everything else is the production code —
shard-local precompute by index offset, fused local passes, Alg. 4 exchange
order, all-reduced observables.  Compared against the single-GPU simulator
and directly against the CPU oracle.  (On an 8-GPU node the same code runs
over NCCL.)"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _mixer(kind, n):
    from paper_2309_04841_b200.mixers import SU2, Mixer

    if kind != "custom":
        return Mixer(kind)
    return Mixer.custom(lambda beta: [SU2(np.cos(beta * (1 + 0.05 * j)), -1j * np.sin(beta * (1 + 0.05 * j)))
                                      for j in range(n)])


def _worker(rank, world, port, n, p, kind, chunk, q, mode="exchange", dev_barrier=True, dtype=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_04841_b200.distributed import ShardedQaoaSimulator
        from paper_2309_04841_b200.problems import labs_terms, portfolio_terms

        rng = np.random.default_rng(11)
        g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
        poly = labs_terms(n) if kind in ("x", "custom") else portfolio_terms(n)
        if kind == "xf":  # float64 costs under the X mixer
            kind = "x"
        sim = ShardedQaoaSimulator(poly, mixer=_mixer(kind, n), chunk_bytes=chunk, global_mode=mode,
                                   device_barrier=dev_barrier, dtype=dtype)
        E = sim.simulate_qaoa(g, b, initial_weight=n // 2 if kind.startswith("xy") else None)
        ov = sim.overlap()
        full = sim.statevector()  # collective gather; must agree with the shards
        lo = rank << (n - (world.bit_length() - 1))
        assert np.array_equal(full[lo:lo + sim.shard.numel()], sim.shard.cpu().numpy())
        q.put((rank, E, ov, sim.exchange_count, sim.shard.cpu().numpy()))
        if mode in ("p2p", "fused"):
            dist.barrier()
            sim.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,p,kind,chunk,mode,dev_barrier",
                         [(16, 3, "x", None, "exchange", True), (17, 2, "x", 1 << 16, "exchange", True),
                          (14, 2, "xy-ring", None, "exchange", True), (16, 3, "x", None, "p2p", True),
                          (19, 2, "x", None, "p2p", False), (15, 2, "custom", None, "p2p", True),
                          (15, 2, "custom", None, "exchange", True),
                          (16, 3, "x", None, "fused", True), (21, 5, "x", None, "fused", True),
                          (15, 2, "custom", None, "fused", True), (14, 3, "xf", None, "fused", True),
                          (14, 2, "xy-ring", None, "fused", True), (15, 1, "xy-complete", None, "fused", True)])
def test_two_process_sharded_matches_single_gpu(n, p, kind, chunk, mode, dev_barrier):
    _run_processes(2, n, p, kind, chunk, mode, dev_barrier)


@pytest.mark.parametrize("n,p,kind", [(15, 3, "x"), (15, 2, "xy-complete"), (16, 2, "custom")])
def test_four_process_fused_matches_single_gpu(n, p, kind):
    """k = 2: four ranks, four IPC-mapped shards, shard sets of the XY passes."""
    _run_processes(4, n, p, kind, None, "fused", True)


def test_two_process_fused_complex64():
    _run_processes(2, 16, 3, "x", None, "fused", True, dtype="complex64")


def _run_processes(world, n, p, kind, chunk, mode, dev_barrier, dtype=None):
    from oracle import oracle as O
    from paper_2309_04841_b200 import Mixer, QaoaSimulator, hamming_weight_state
    from paper_2309_04841_b200.problems import labs_terms, portfolio_terms

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, p, kind, chunk, q, mode, dev_barrier, dtype))
             for r in range(world)]
    for pr in procs:
        pr.start()
    out = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    rng = np.random.default_rng(11)
    g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
    poly = labs_terms(n) if kind in ("x", "custom") else portfolio_terms(n)
    kind = "x" if kind == "xf" else kind
    sim = QaoaSimulator(terms=poly, mixer=_mixer(kind, n))
    init = hamming_weight_state(n, n // 2) if kind.startswith("xy") else None
    res = sim.simulate_qaoa(g, b, initial=init)
    full = np.concatenate([o[4] for o in out])
    tol = 1e-12 if dtype is None else 1e-4 * np.abs(res.state).max()  # complex64: the fp32 tolerance
    np.testing.assert_allclose(full, res.state, rtol=0, atol=tol)
    # and directly against the CPU oracle (not only CUDA against CUDA)
    costs = sim.get_cost_diagonal()
    factory = None
    if kind == "custom":
        mixer = _mixer(kind, n)
        factory = lambda beta: [(u.a, u.b) for u in mixer.su2_factory(beta)]  # noqa: E731
    ref = O.simulate(costs, g, b, kind, init, su2_factory=factory)
    otol = 1e-10 if dtype is None else 1e-4
    np.testing.assert_allclose(full, ref, rtol=0, atol=otol * np.abs(ref).max())
    e_ref = O.expectation(ref, costs)
    for rank, E, ov, ex, _ in out:
        assert E == pytest.approx(sim.get_expectation(res), rel=1e-10 if dtype is None else 1e-4, abs=1e-12)
        assert E == pytest.approx(e_ref, rel=otol, abs=1e-12)
        assert ov == pytest.approx(sim.get_overlap(res), abs=1e-12 if dtype is None else 1e-4)
        if kind in ("x", "custom"):
            assert ex == 2 * p  # Alg. 4: two exchanges per layer
