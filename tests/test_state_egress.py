"""State egress: save_state / load_state file layout
(reference statevec.py:114-123, tests/test_statevec.py:171-184), destructive
probabilities (statevec.py:81-91, tests/test_statevec.py:157-163) and the
live-result contract of QaoaSimulator (qaoa.py:63-68: the objective follows
in-place updates of the result's state)."""

import numpy as np
import pytest

from paper_2309_04841_b200.statevec import load_state, save_state


def _random_state(rng, n):
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return psi / np.linalg.norm(psi)


def test_state_file_round_trip(tmp_path):
    state = _random_state(np.random.default_rng(7), 3)
    path = tmp_path / "state.bin"
    save_state(state, str(path))
    np.testing.assert_array_equal(load_state(str(path)), state)


def test_state_file_layout_is_interleaved_little_endian(tmp_path):
    state = np.array([1.0 + 2.0j, -0.5 + 0.25j])
    path = tmp_path / "state.bin"
    save_state(state, str(path))
    np.testing.assert_array_equal(np.fromfile(str(path), dtype="<f8"), [1.0, 2.0, -0.5, 0.25])


def test_load_state_rejects_non_power_of_two(tmp_path):
    path = tmp_path / "bad.bin"
    np.zeros(3, dtype="<c16").tofile(str(path))
    with pytest.raises(ValueError, match="power of two"):
        load_state(str(path))


@pytest.mark.gpu
def test_device_state_file_round_trip(tmp_path):
    import torch

    state = _random_state(np.random.default_rng(8), 13)
    dev = torch.from_numpy(state).cuda()
    path = tmp_path / "dev.bin"
    save_state(dev, str(path))
    np.testing.assert_array_equal(load_state(str(path)), state)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [10, 16])
def test_simulator_destructive_probabilities_is_a_view_of_the_state(n):
    from paper_2309_04841_b200 import QaoaSimulator, labs_terms

    sim = QaoaSimulator(terms=labs_terms(n))
    res = sim.simulate_qaoa([0.2, 0.4], [0.3, 0.1])
    expected = np.abs(res.state.copy()) ** 2
    probs = sim.get_probabilities(res, preserve_state=False)
    np.testing.assert_allclose(probs, expected, rtol=0, atol=1e-15)
    assert probs.base is res.state  # a view of the squared state, as the reference's state.real
    np.testing.assert_allclose(res.state.imag, 0.0, atol=0)
    np.testing.assert_allclose(res.state_device.cpu().numpy().real, expected, rtol=0, atol=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [10, 16])
def test_result_objective_follows_in_place_updates(n):
    """The fused last pass caches the objective; an in-place operation on the
    result's state (here the operator-layer phase and mixer) retires it."""
    from paper_2309_04841_b200 import QaoaSimulator, labs_terms, statevec
    from paper_2309_04841_b200.mixers import rx_layer

    from oracle import oracle as O

    sim = QaoaSimulator(terms=labs_terms(n))
    res = sim.simulate_qaoa([0.2], [0.3])
    e0 = sim.get_expectation(res)
    host0 = res.state.copy()
    costs = sim.get_cost_diagonal()
    statevec.apply_phase(res.state_device, costs, 0.7)
    rx_layer(res.state_device, 0.45)
    ref = host0.copy()
    O.apply_phase(ref, np.array(costs), 0.7)
    O.rx_layer(ref, 0.45)
    np.testing.assert_allclose(res.state, ref, rtol=0, atol=1e-12)  # host copy refreshed
    e1 = sim.get_expectation(res)
    assert e1 == pytest.approx(O.expectation(ref, np.array(costs)), rel=1e-12)
    assert e1 != pytest.approx(e0, rel=1e-6)


@pytest.mark.gpu
def test_reused_buffer_retires_the_previous_result():
    from paper_2309_04841_b200 import QaoaSimulator, labs_terms

    sim = QaoaSimulator(terms=labs_terms(14))
    r1 = sim.simulate_qaoa([0.2], [0.3], reuse_buffer=True)
    r2 = sim.simulate_qaoa([0.5], [0.1], reuse_buffer=True)
    # r1's buffer now holds r2's state: its objective is recomputed from it, not stale
    assert sim.get_expectation(r1) == pytest.approx(sim.get_expectation(r2), rel=1e-12)


@pytest.mark.gpu
def test_costs_from_array_rejects_non_power_of_two():
    from paper_2309_04841_b200 import QaoaSimulator

    with pytest.raises(ValueError, match="power of two"):
        QaoaSimulator(costs=np.zeros(12))
