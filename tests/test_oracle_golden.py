"""Pin the CPU oracle (oracle/) against vectors produced by the reference itself
(tests/golden/golden.npz, written by scripts/gen_golden.py from
/root/reference/pkg/src).  CPU only."""

import numpy as np
import pytest

from _helpers import golden_terms
from oracle import oracle as O

DIAGS = ["labs8", "labs12", "labs14", "tri", "cubic12", "maxcut26sub14", "rand5", "rand8", "rand10", "port8",
         "port12"]


@pytest.mark.parametrize("name", DIAGS)
def test_diagonal_bit_exact(golden, name):
    # reference _kernels.accumulate_terms vs the C restatement: identical bits,
    # float weights included (same per-element left-to-right accumulation)
    n, pairs = golden_terms(golden, name)
    got = O.precompute_cost_vector(n, pairs)
    np.testing.assert_array_equal(got.view(np.uint64), golden[f"diag/{name}"].view(np.uint64))


def test_diagonal_sharded_slices(golden):
    n, pairs = golden_terms(golden, "labs12")
    full = golden["diag/labs12"]
    for r in range(4):
        part = O.precompute_cost_vector(n, pairs, base=r * 1024, size=1024)
        np.testing.assert_array_equal(part, full[r * 1024:(r + 1) * 1024])


def test_known_answers():
    # reference tests/test_terms.py:102-120
    np.testing.assert_array_equal(O.precompute_cost_vector(2, [(1.0, (0, 1))]), [1, -1, -1, 1])
    np.testing.assert_array_equal(O.precompute_cost_vector(3, []), np.zeros(8))
    tri = [(0.5, (0, 1)), (0.5, (0, 2)), (0.5, (1, 2)), (-1.5, ())]
    np.testing.assert_array_equal(O.precompute_cost_vector(3, tri), [0, -2, -2, -2, -2, -2, -2, 0])


def test_labs_identity():
    # reference tests/test_problems.py:114-121: 2 f + n(n-1)/2 == E exhaustively
    for n in range(2, 11):
        c = O.precompute_cost_vector(n, O.labs_terms(n))
        for k in range(1 << n):
            assert 2 * c[k] + n * (n - 1) // 2 == O.labs_energy(k, n)


SIMS = ["labs8_x_p3", "labs12_x_p4", "labs14_x_p3", "rand5_x_p2", "rand10_x_p5", "cubic12_x_p6",
        "maxcut26sub14_x_p2", "port8_ring_p2", "port8_complete_p2", "port12_ring_p2", "port12_complete_p1",
        "labs8_custom_p2"]


def _poly_of(case):
    return case.split("_")[0]


@pytest.mark.parametrize("case", SIMS)
def test_simulation_matches_reference(golden, case):
    name = _poly_of(case)
    n, pairs = golden_terms(golden, name)
    costs = golden[f"diag/{name}"]
    g, b = golden[f"sim/{case}/gammas"], golden[f"sim/{case}/betas"]
    kind = {"x": "x", "ring": "xy-ring", "complete": "xy-complete", "custom": "custom"}[case.split("_")[1]]
    initial = O.hamming_weight_state(n, {8: 4, 12: 6}[n]) if kind.startswith("xy") else None
    fac = (lambda bb: [(np.cos(bb), np.sin(bb))] * n) if kind == "custom" else None
    state = O.simulate(costs, g, b, kind, initial, fac)
    ref = golden[f"sim/{case}/state"]
    np.testing.assert_allclose(state, ref, rtol=0, atol=1e-13)
    assert O.expectation(state, costs) == pytest.approx(float(golden[f"sim/{case}/E"]), rel=1e-12, abs=1e-12)
    assert O.overlap(state, costs) == pytest.approx(float(golden[f"sim/{case}/overlap"]), abs=1e-12)


def test_exchange_matches_reference(golden):
    st = golden["exchange/n6K4/in"].copy()
    shards = [st[r * 16:(r + 1) * 16].copy() for r in range(4)]
    O.exchange(shards)
    np.testing.assert_array_equal(np.concatenate(shards), golden["exchange/n6K4/out"])
    np.testing.assert_array_equal(O.transpose_oracle(golden["exchange/n6K4/in"], 2), golden["exchange/n6K4/out"])


def test_distributed_reference_equals_single_node(golden):
    # the reference's sharded run (K=4) equals the single-node oracle evolution
    n, pairs = golden_terms(golden, "labs8")
    costs = golden["diag/labs8"]
    st = O.simulate(costs, golden["dist/labs8_K4/gammas"], golden["dist/labs8_K4/betas"])
    np.testing.assert_allclose(st, golden["dist/labs8_K4/state"], atol=1e-12)
    assert int(golden["dist/labs8_K4/exchanges"]) == 2 * 3


def test_phase_goldens():
    # reference tests/test_statevec.py:70-80
    st = O.uniform_state(2)
    O.apply_phase(st, np.ones(4), np.pi)
    np.testing.assert_allclose(st, np.full(4, -0.5), atol=1e-15)
    st = O.uniform_state(2)
    O.apply_phase(st, np.array([1.0, -1.0, -1.0, 1.0]), np.pi / 2)
    np.testing.assert_allclose(st, [-0.5j, 0.5j, 0.5j, -0.5j], atol=1e-15)


def test_rx_goldens():
    # reference tests/test_mixers.py:167-180: |+>^n is an eigenstate; beta = pi/2 flips every bit
    n = 5
    st = O.uniform_state(n)
    O.rx_layer(st, 0.37)
    np.testing.assert_allclose(np.abs(st), np.abs(O.uniform_state(n)), atol=1e-14)
    st = np.zeros(1 << n, dtype=np.complex128)
    st[0] = 1.0
    O.rx_layer(st, np.pi / 2)
    assert abs(st[-1] - (-1j) ** n) < 1e-14


def test_edge_orders():
    # reference tests/test_mixers.py:244-251
    assert O.ring_edges(5) == [(0, 1), (2, 3), (1, 2), (3, 4), (4, 0)]
    assert O.ring_edges(2) == [(0, 1)]
    assert O.complete_edges(4) == [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
