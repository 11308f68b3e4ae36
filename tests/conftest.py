import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


import pytest  # noqa: E402


@pytest.fixture(autouse=True)
def _release_gpu_memory():
    """After every test: close the EpMoE contexts it left open and drop the last failure's
    traceback (pytest keeps it in sys.last_traceback, and its frames hold the test's tensors), so a
    failed full-size test does not starve the next one of device memory."""
    yield
    if "torch" not in sys.modules or "paper_2604_19241_b200.moe" not in sys.modules:
        return
    import gc
    torch = sys.modules["torch"]
    moe = sys.modules["paper_2604_19241_b200.moe"]
    for ctx in moe.live_contexts():
        ctx.close()
    sys.last_traceback = sys.last_value = sys.last_type = None
    if hasattr(sys, "last_exc"):
        sys.last_exc = None
    gc.collect()
    if torch.cuda.is_available():
        torch.cuda.empty_cache()
