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
    # the native libraries are build artefacts (git-ignored): build them if missing or stale
    # (nvcc cross-compiles sm_100a without a GPU; the oracle is plain gcc)
    from paper_2309_04841_b200 import _build

    if _build._stale():
        _build.build()
    from oracle import oracle as O

    O.build()


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
