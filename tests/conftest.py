import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not gpu_available():
        pytest.skip("no GPU in this container")
    import paper_1803_11036_b200 as P
    assert P.device_count() >= 1
    return P


@pytest.fixture(autouse=True)
def _checked_build_clean(request):
    """Under SSPD_CHECKED_ASSERT=1 (tests/test_gpu_checked.py runs the GPU
    suites on lib/libsspd_cuda_checked.so): after every GPU test, no device
    bounds check or window-ring invariant may have failed."""
    yield
    if os.environ.get("SSPD_CHECKED_ASSERT") != "1" or "gpu" not in request.keywords:
        return
    import paper_1803_11036_b200 as P
    line, n = P.checked_status(0, reset=True)
    assert n == 0, f"{n} device check failure(s), first at kernels.cuh:{line}"
