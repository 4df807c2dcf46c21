"""Parity at the BASELINE configurations' full sizes (n = 22 / 26) against
fingerprints of the reference's own outputs (tests/golden/golden_large.npz):
bit-exact cost diagonal (SHA-256), objective and overlap to 1e-10, 4096
sampled amplitudes and 1024 block norms to 1e-10 absolute (fp64)."""

import numpy as np
import pytest

from _large import CASES, check_fingerprint
from paper_2309_04841_b200 import Mixer, QaoaSimulator, hamming_weight_state

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", list(CASES))
def test_full_size_matches_reference(golden_large, name):
    make, kind, hw = CASES[name]
    poly = make()
    sim = QaoaSimulator(terms=poly, mixer=Mixer(kind))
    initial = hamming_weight_state(poly.n, hw) if hw is not None else None
    res = sim.simulate_qaoa(golden_large[f"{name}/gammas"], golden_large[f"{name}/betas"], initial=initial)
    E = sim.get_expectation(res)
    ov = sim.get_overlap(res)
    check_fingerprint(golden_large, name, sim.get_cost_diagonal(), sim.get_statevector(res), E, ov)


def test_full_size_objective_loop_is_stable(golden_large):
    """The objective of the headline configuration is reproducible call to call
    (deterministic reductions: identical bits every evaluation)."""
    make, kind, _ = CASES["labs26_x_p10"]
    sim = QaoaSimulator(terms=make())
    g, b = golden_large["labs26_x_p10/gammas"], golden_large["labs26_x_p10/betas"]
    vals = {sim.get_expectation(sim.simulate_qaoa(g, b, reuse_buffer=True)) for _ in range(3)}
    assert len(vals) == 1


@pytest.mark.parametrize("name,K", [("labs26_x_p10", 8), ("maxcut26_x_p6", 4), ("port22_complete_p1", 2),
                                    ("port26_ring_p1", 8)])
def test_full_size_sharded_program_matches_reference(golden_large, name, K):
    """The fused sharded program (in-process, K shard views; its spanning passes are
    the multi-GPU kernels) against the reference's own full-size outputs."""
    from paper_2309_04841_b200 import QaoaParams
    from paper_2309_04841_b200.distributed import simulate_qaoa_distributed

    make, kind, hw = CASES[name]
    poly = make()
    initial = hamming_weight_state(poly.n, hw) if hw is not None else None
    params = QaoaParams(tuple(golden_large[f"{name}/gammas"]), tuple(golden_large[f"{name}/betas"]))
    res = simulate_qaoa_distributed(poly, params, K, mixer=Mixer(kind), initial=initial)
    check_fingerprint(golden_large, name, res.costs, res.statevector(), res.expectation(), res.overlap())


def test_full_size_complex64_labs30(golden_large):
    """complex64 at the reference's size limit (LABS n = 30, p = 3) against its own outputs, fp32 tolerance."""
    name = "labs30_x_p3"
    make, _, _ = CASES[name]
    sim = QaoaSimulator(terms=make(), dtype="complex64")
    res = sim.simulate_qaoa(golden_large[f"{name}/gammas"], golden_large[f"{name}/betas"])
    e_ref = float(golden_large[f"{name}/E"])
    assert abs(sim.get_expectation(res) - e_ref) <= 1e-4 * max(1.0, abs(e_ref))
    state = sim.get_statevector(res)
    amp = golden_large[f"{name}/amp"]
    np.testing.assert_allclose(state[golden_large[f"{name}/idx"]], amp, rtol=0, atol=1e-4 * np.abs(amp).max())
