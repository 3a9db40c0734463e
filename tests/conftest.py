import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA extension")
    config.addinivalue_line("markers", "slow: long-running (large shapes)")


@pytest.fixture(scope="session")
def port():
    """The C restatement oracle (checker only)."""
    from oracle import pyoracle

    return pyoracle.load("port")


@pytest.fixture(scope="session")
def ref():
    """The reference itself, compiled from its sources (oracle/_ref); skipped
    where neither the sources nor the prebuilt library exist."""
    from oracle import pyoracle

    if not pyoracle.available("ref"):
        pytest.skip("reference library not available here")
    return pyoracle.load("ref")


@pytest.fixture(scope="session")
def msvd():
    """The CUDA extension, built in-tree if absent (fails loudly, never falls back)."""
    from paper_2602_16797_b200 import minsvd

    if not os.path.exists(minsvd.LIB_PATH):
        minsvd.build()
    minsvd.lib()
    return minsvd


@pytest.fixture(scope="session")
def cuda(msvd):
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    cap = torch.cuda.get_device_capability(0)
    assert cap[0] == 10, f"expected sm_100 (B200), got sm_{cap[0]}{cap[1]}"
    return torch.device("cuda:0")
