import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200, sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _ensure_oracle():
    from oracle import pyoracle
    if not os.path.exists(pyoracle.PORT_SO):
        pyoracle.build(ref=os.path.isdir("/root/reference/proj/include"))
    return pyoracle


@pytest.fixture(scope="session")
def pyoracle():
    return _ensure_oracle()


@pytest.fixture(scope="session")
def port(pyoracle):
    """The plain-C restatement (always available)."""
    return pyoracle.Oracle("port")


@pytest.fixture(scope="session")
def ref(pyoracle):
    """The compiled, unmodified reference (oracle/_ref), when present."""
    if not os.path.exists(pyoracle.REF_SO):
        pytest.skip("oracle/_ref/libedx_ref.so not built (reference sources absent)")
    return pyoracle.Oracle("reference")


@pytest.fixture(scope="session")
def oracle(pyoracle):
    """Best available checker: the compiled reference, else the restatement."""
    if os.path.exists(pyoracle.REF_SO):
        return pyoracle.Oracle("reference")
    return pyoracle.Oracle("port")


@pytest.fixture(scope="session")
def edx():
    import paper_2512_21615_b200 as edx
    return edx


@pytest.fixture(scope="session")
def gpu(edx):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected on a host without CUDA")
    return edx
