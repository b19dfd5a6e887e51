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


def _reload_tuning():
    try:
        import paper_2402_02750_b200 as kb
        if os.path.exists(kb.LIB_PATH):
            kb.reload_tuning()
    except Exception:
        pass


@pytest.fixture(autouse=True)
def _kivi_tuning(monkeypatch):
    """The library reads its KIVI_* routing knobs once (kivi_reload_tuning
    re-reads them): reload at the start of every test (the previous test's
    monkeypatch has been undone) and on every monkeypatched KIVI_* change."""
    _reload_tuning()
    orig_set, orig_del = monkeypatch.setenv, monkeypatch.delenv

    def setenv(name, value, prepend=None):
        orig_set(name, value, prepend)
        if name.startswith("KIVI_"):
            _reload_tuning()

    def delenv(name, raising=True):
        orig_del(name, raising)
        if name.startswith("KIVI_"):
            _reload_tuning()

    monkeypatch.setenv = setenv
    monkeypatch.delenv = delenv
    yield


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
