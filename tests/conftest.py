import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; parity tests through the C ABI")


@pytest.fixture(scope="session")
def port():
    """Our C restatement of the reference (oracle/libtgs_oracle.so), built on demand."""
    from oracle import oracle
    if not os.path.exists(oracle.PORT_SO):
        oracle.build(ref=False)
    return oracle.Port()


@pytest.fixture(scope="session")
def ref():
    """The reference compiled from its own sources (oracle/_ref), when available."""
    from oracle import oracle
    if not oracle.Ref.available():
        if os.path.isdir(oracle.REF_SRC):
            oracle.build(ref=True)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    return oracle.Ref()


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    from tests.cases import CASES
    out = {}
    for name in CASES:
        out[name] = dict(np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz")))
    return out
