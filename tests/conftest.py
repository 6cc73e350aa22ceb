import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libvsdock.so")


def _has_gpu():
    try:
        from paper_2110_11644_b200 import native
        return native.lib().vs_device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu_ctx():
    if not _has_gpu():
        pytest.fail("GPU test selected but no CUDA device / libvsdock.so is usable (no fallback exists)")
    from paper_2110_11644_b200 import api
    return api.default_context(0)


@pytest.fixture(scope="session")
def port():
    from oracle import Oracle
    return Oracle("port", trig=0)


@pytest.fixture(scope="session")
def port_cr():
    """The oracle with the GPU's correctly rounded torsion trig (bit-parity checker)."""
    from oracle import Oracle
    return Oracle("port", trig=1)


def oracle_kinds():
    from oracle import available
    kinds = ["port"]
    if available("ref"):
        kinds.append("ref")
    return kinds
