"""Pin the CPU oracle against the reference at full size (n = 22 LABS, n = 26
MaxCut of BASELINE config 2): bit-exact diagonal, objective, overlap and
state fingerprints (tests/golden/golden_large.npz).  CPU only, ~20 s."""

import numpy as np
import pytest

from _large import CASES, check_fingerprint
from oracle import oracle as O


def _pairs(poly):
    return [(t.weight, t.support) for t in poly.terms]


@pytest.mark.parametrize("name", ["labs22_x_p4", "maxcut26_x_p6"])
def test_oracle_matches_reference_full_size(golden_large, name):
    make, kind, _ = CASES[name]
    poly = make()
    costs = O.precompute_cost_vector(poly.n, _pairs(poly))
    state = O.simulate(costs, golden_large[f"{name}/gammas"], golden_large[f"{name}/betas"], kind)
    check_fingerprint(golden_large, name, costs, state, O.expectation(state, costs), O.overlap(state, costs))
