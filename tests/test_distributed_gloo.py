"""Multi-process sharding (ShardedQaoaSimulator, one rank per GPU in
production) on CPU: world size 2 over gloo, the shard-local work done by a
test-only backend on the oracle (oracle/, the checker), the orchestration —
global-qubit split, Alg. 4 exchange order, chunked exchange, exchange counts,
scalar reductions — is the product code (paper_2309_04841_b200/distributed.py).
Reference behaviour: distributed.py:103-153, 228-252; tests/test_distributed.py."""

import os
import socket
from math import comb, sqrt

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


class OracleOps:
    """Shard-local operations for ShardedQaoaSimulator on host tensors (test only)."""

    def fits(self, n_local, bytes_per_amp):
        return True

    def fits_bytes(self, nbytes):
        return True

    def precompute(self, poly, base, n_local, compact, keep_f64):
        pairs = [(t.weight, t.support) for t in poly.terms]
        return O.precompute_cost_vector(poly.n, pairs, base=base, size=1 << n_local)

    def empty(self, n_local):
        return torch.empty(1 << n_local, dtype=torch.complex128)

    def uniform(self, n, n_local):
        return torch.full((1 << n_local,), 1.0 / sqrt(2.0 ** n), dtype=torch.complex128)

    def hamming(self, n, weight, base, n_local):
        idx = np.arange(base, base + (1 << n_local), dtype=np.int64)
        pop = np.array([bin(int(i)).count("1") for i in idx])
        return torch.from_numpy(np.where(pop == weight, 1.0 / sqrt(comb(n, weight)), 0.0).astype(np.complex128))

    def program(self, psi, n_local, kind, layers, costs, init=False, init_amp=0.0, su2=None):
        assert kind in ("x", "custom")
        st = psi.numpy()
        if init:
            st[:] = init_amp
        for li, (g, b, ph, lo, hi) in enumerate(layers):
            if ph and g != 0.0:
                O.apply_phase(st, costs, g)
            for q in range(lo, hi):
                if kind == "x":
                    a, bb = O.rx_coeffs(b)
                else:
                    c = su2[li][q]
                    a, bb = complex(c[0], c[1]), complex(c[2], c[3])
                O.su2_on_pairs(st, a, bb, q)

    def xy(self, psi, beta, lo, hi):
        O.xy_on_pairs(psi.numpy(), float(np.cos(beta)), float(np.sin(beta)), lo, hi)

    def swap(self, psi, lo, hi):
        O.swap_bits(psi.numpy(), lo, hi)

    def expectation(self, psi, costs):
        return torch.tensor([O.expectation(psi.numpy(), costs)], dtype=torch.float64)

    def min_cost(self, costs):
        return torch.tensor([float(costs.min())], dtype=torch.float64)

    def masked_probability(self, psi, costs, cutoff):
        p = np.abs(psi.numpy()) ** 2
        return torch.tensor([float(p[costs <= cutoff].sum())], dtype=torch.float64)


def _worker(rank, world, port, n, p, chunk, q, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_04841_b200 import instrumentation
        from paper_2309_04841_b200.distributed import ShardedQaoaSimulator
        from paper_2309_04841_b200.problems import labs_terms

        rng = np.random.default_rng(5)
        g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
        sim = ShardedQaoaSimulator(labs_terms(n), local_ops=OracleOps(), chunk_bytes=chunk)
        instrumentation.reset()
        E = sim.simulate_qaoa(g, b)
        ov = sim.overlap()
        full = sim.statevector()  # gather of the shards on every rank
        sim.save_shard(os.path.join(outdir, f"shard{rank}.bin"), chunk_bytes=1024)  # streamed egress
        q.put((rank, E, ov, sim.exchange_count, instrumentation.get("exchange"), full if rank == 0 else None))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n,p,chunk", [(10, 3, None), (11, 2, 4096)])
def test_sharded_world2_matches_single_node(n, p, chunk, tmp_path):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, p, chunk, q, str(tmp_path))) for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    out.sort(key=lambda t: t[0])
    rng = np.random.default_rng(5)
    g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
    costs = O.precompute_cost_vector(n, O.labs_terms(n))
    ref = O.simulate(costs, g, b)
    e_ref, ov_ref = O.expectation(ref, costs), O.overlap(ref, costs)
    for rank, E, ov, ex, ex_counter, state in out:
        assert E == pytest.approx(e_ref, rel=1e-12, abs=1e-12)  # all-reduced on every rank
        assert ov == pytest.approx(ov_ref, abs=1e-12)
        assert ex == 2 * p and ex_counter == 2 * p  # Alg. 4: two exchanges per X layer
    np.testing.assert_allclose(out[0][5], ref, rtol=0, atol=1e-12)
    # save_shard files in rank order = the reference's save_state file of the whole state
    whole = tmp_path / "whole.bin"
    with open(whole, "wb") as f:
        for r in range(world):
            f.write((tmp_path / f"shard{r}.bin").read_bytes())
    from paper_2309_04841_b200.statevec import load_state

    np.testing.assert_array_equal(load_state(str(whole)), out[0][5])


def _xy_worker(rank, world, port, n, p, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_04841_b200.distributed import ShardedQaoaSimulator
        from paper_2309_04841_b200.problems import portfolio_terms

        rng = np.random.default_rng(7)
        g, b = rng.uniform(-1, 1, p), rng.uniform(-1, 1, p)
        sim = ShardedQaoaSimulator(portfolio_terms(n), mixer=kind, local_ops=OracleOps())
        E = sim.simulate_qaoa(g, b, initial_weight=n // 2)
        shards = [torch.empty_like(sim.shard) for _ in range(world)]
        dist.all_gather(shards, sim.shard)
        q.put((rank, E, sim.exchange_count, torch.cat(shards).numpy() if rank == 0 else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["xy-ring", "xy-complete"])
def test_sharded_xy_world2_matches_single_node(kind):
    """XY mixers over 2 ranks (reference distributed.py:160-207 algorithm: park +
    exchange for pairs touching the global qubit) equal the single-node oracle."""
    n, p, world = 8, 2, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xy_worker, args=(r, world, port, n, p, kind, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    rng = np.random.default_rng(7)
    g, b = rng.uniform(-1, 1, p), rng.uniform(-1, 1, p)
    from paper_2309_04841_b200.problems import portfolio_terms

    poly = portfolio_terms(n)
    costs = O.precompute_cost_vector(n, [(t.weight, t.support) for t in poly.terms])
    ref = O.simulate(costs, g, b, kind, O.hamming_weight_state(n, n // 2))
    edges = O.ring_edges(n) if kind == "xy-ring" else O.complete_edges(n)
    assert out[0][2] == p * 2 * sum(1 for i, j in edges if max(i, j) >= n - 1)  # 2 exchanges per global pair
    for rank, E, ex, state in out:
        assert E == pytest.approx(O.expectation(ref, costs), rel=1e-12, abs=1e-12)
    np.testing.assert_allclose(out[0][3], ref, rtol=0, atol=1e-12)


def _custom_worker(rank, world, port, n, p, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_04841_b200.distributed import ShardedQaoaSimulator
        from paper_2309_04841_b200.mixers import SU2, Mixer
        from paper_2309_04841_b200.problems import labs_terms

        rng = np.random.default_rng(3)
        g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
        mixer = Mixer.custom(lambda beta: [SU2(np.cos(beta + 0.1 * j), np.sin(beta + 0.1 * j)) for j in range(n)])
        sim = ShardedQaoaSimulator(labs_terms(n), mixer=mixer, local_ops=OracleOps())
        E = sim.simulate_qaoa(g, b)
        shards = [torch.empty_like(sim.shard) for _ in range(world)]
        dist.all_gather(shards, sim.shard)
        q.put((rank, E, sim.exchange_count, torch.cat(shards).numpy() if rank == 0 else None))
    finally:
        dist.destroy_process_group()


def test_sharded_custom_mixer_world2():
    """Custom per-qubit SU(2) mixers over 2 ranks (Alg. 4 with arbitrary gates:
    distributed.py:137-153)."""
    n, p, world = 9, 2, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_custom_worker, args=(r, world, port, n, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    rng = np.random.default_rng(3)
    g, b = rng.uniform(0, 1, p), rng.uniform(0, 1, p)
    costs = O.precompute_cost_vector(n, O.labs_terms(n))
    factory = lambda beta: [(complex(np.cos(beta + 0.1 * j)), complex(np.sin(beta + 0.1 * j))) for j in range(n)]
    st = O.uniform_state(n)
    for gg, bb in zip(g, b):
        O.apply_phase(st, costs, gg)
        for qb, (a, bc) in enumerate(factory(bb)):
            O.su2_on_pairs(st, a, bc, qb)
    np.testing.assert_allclose(out[0][3], st, rtol=0, atol=1e-12)
    assert out[0][2] == 2 * p
