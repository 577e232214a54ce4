import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def port():
    import oracle

    return oracle.Port()


@pytest.fixture(scope="session")
def builder():
    if not gpu_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_1709_07781_b200 import ndx

    return ndx.WahBuilder(1 << 16)


@pytest.fixture(scope="session")
def prims():
    if not gpu_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_1709_07781_b200 import ndx

    return ndx.Primitives()
