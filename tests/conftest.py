import os
import sys

import hypothesis
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

hypothesis.settings.register_profile("default", deadline=None, max_examples=50, derandomize=True)
hypothesis.settings.load_profile("default")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    path = os.path.join(ROOT, "tests", "golden", "golden.npz")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_large():
    """Full-size fingerprints of the reference's outputs (scripts/gen_golden_large.py)."""
    import numpy as np

    path = os.path.join(ROOT, "tests", "golden", "golden_large.npz")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}
