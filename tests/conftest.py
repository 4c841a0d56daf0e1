import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture
def rng():
    # same seed as the reference's tests/conftest.py:16-18
    return np.random.default_rng(20260814)


def random_dominant_bands(n, seed, ratio=0.3):
    """Reference tests/conftest.py:7-13: b in [2,3), a,c in ratio*[-1,1)."""
    r = np.random.default_rng(seed)
    b = 2.0 + r.random(n)
    a = ratio * (2.0 * r.random(n) - 1.0)
    c = ratio * (2.0 * r.random(n) - 1.0)
    return a, b, c


def golden_run(g, tag):
    """Unpack one run_distd2 golden case."""
    st = g[f"run_{tag}_stencil"]
    return dict(lower=g[f"run_{tag}_lower"], diag=g[f"run_{tag}_diag"],
                upper=g[f"run_{tag}_upper"],
                periodic=bool(g[f"run_{tag}_periodic"]),
                stencil=None if st.shape[0] == 0 else st,
                field=g[f"run_{tag}_field"],
                sizes=tuple(int(s) for s in g[f"run_{tag}_sizes"]),
                out=g[f"run_{tag}_out"])
