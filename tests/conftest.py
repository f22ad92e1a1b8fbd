import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running case")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(HERE, "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_arrays():
    return dict(np.load(os.path.join(HERE, "golden", "golden.npz")))


@pytest.fixture(scope="session")
def product():
    import impls
    return impls.product()


@pytest.fixture(scope="session")
def port():
    import impls
    return impls.port()


@pytest.fixture(scope="session")
def reference():
    import impls
    if not impls.have_reference():
        pytest.skip("oracle/_ref/libsplbref.so not built")
    return impls.reference()
