"""Shared fixtures.  GPU tests are marked @pytest.mark.gpu and call the CUDA path through the C ABI;
everything else runs on CPU (oracle pins, host logic, ABI export checks, gloo multi-process)."""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


@pytest.fixture(scope="session")
def port():
    from oracle.pyoracle import Oracle, build
    build()
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference behind the oracle ABI; skipped when oracle/_ref was never built."""
    from oracle.pyoracle import Oracle, build
    build()
    if not Oracle.available("reference"):
        pytest.skip("oracle/_ref not built (no reference tree on this machine)")
    return Oracle("reference")


def load_golden(name):
    z = np.load(GOLDEN / name, allow_pickle=False)
    return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden():
    return load_golden
