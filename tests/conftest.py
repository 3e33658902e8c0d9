import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libscreloc_gpu.so")
    config.addinivalue_line("markers", "slow: long-running (CPU oracle end-to-end)")


@pytest.fixture(scope="session")
def oracle():
    import oracle_ffi

    return oracle_ffi.get()


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu_device():
    if not gpu_available():
        pytest.fail("GPU test run without a GPU: the product has no CPU fallback")
    from paper_1810_12163_b200 import build

    build.build()
    import paper_1810_12163_b200 as P

    return P.Device(0)
