import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libmonet_b200.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2010_14501_b200 import _native
    assert _native.lib().device_check() == 0, "not an sm_100 device"
    return torch.device("cuda:0")


@pytest.fixture(autouse=True)
def _cpu_threads(request):
    """CPU tests replay small networks: torch's intra-op thread pool only adds fork/spin
    overhead there (a 2x16x32x32 float64 conv: 0.6 ms on one thread, 0.26 s on eight when
    the host is busy), so they run single-threaded; GPU tests keep the pool (the headline
    parity test replays ResNet-50 b184 on the CPU oracle)."""
    if request.node.get_closest_marker("gpu"):
        yield
        return
    import torch
    n = torch.get_num_threads()
    torch.set_num_threads(1)
    try:
        yield
    finally:
        torch.set_num_threads(n)
