import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA sm_100) device")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _have_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the native libraries if they are missing (the driver normally runs build())."""
    lib = os.path.join(ROOT, "paper_1911_06001_b200", "lib")
    need = not (os.path.exists(os.path.join(lib, "libvxa.so")) and os.path.exists(os.path.join(lib, "libvoxanim.so")))
    need_ref = os.path.isdir("/root/reference/proj") and not os.path.exists(
        os.path.join(ROOT, "oracle", "_ref", "libvoxanim_ref.so"))
    if need or need_ref:
        import __graft_entry__

        __graft_entry__.build()
    yield


@pytest.fixture(scope="session")
def gpu():
    if not _have_gpu():
        pytest.skip("no CUDA device")
    return True
