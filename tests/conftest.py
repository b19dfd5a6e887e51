import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


# The library routes small unit counts (U * l / 256 < 4 * SMs) through small
# items only (kivi_b200.cu, KIVI_SMALL_ITEMS).  Parity tests use a few units,
# so they pin the body + tail split by default; the small-item route has its
# own parametrised cases (test_gpu_parity.py, item_policy).
os.environ.setdefault("KIVI_SMALL_ITEMS", "0")
os.environ.setdefault("KIVI_SMALL_FUSED", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
