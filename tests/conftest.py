import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: full-size configs")


def rel_err(got, want):
    """The reference's tolerance convention (tests/testutil.hpp:14-20)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    den = np.maximum(1.0, np.maximum(np.abs(got), np.abs(want)))
    return np.abs(got - want) / den


@pytest.fixture(scope="session")
def orc():
    import oracle as O
    return O.restatement()


@pytest.fixture(scope="session")
def ref():
    import oracle as O
    r = O.reference()
    if r is None:
        pytest.skip("reference build oracle/_ref absent")
    return r


@pytest.fixture(scope="session")
def capi():
    from paper_2605_24290_b200 import capi as c
    return c


@pytest.fixture(scope="session")
def ctx(capi):
    return capi.Context(0)
