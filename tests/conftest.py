"""Test configuration: markers, import paths, in-tree build of the product library."""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu() -> bool:
    try:
        from paper_2406_03488_b200 import _capi
        import ctypes
        n = ctypes.c_int32(0)
        _capi.lib().sp_cuda_device_count(ctypes.byref(n))
        return n.value > 0
    except Exception:
        return False


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    from paper_2406_03488_b200 import _capi, build
    if not _capi.LIB_PATH.exists() and os.environ.get("SEQPIPE_NO_BUILD") != "1":
        build.build()
    yield


@pytest.fixture(scope="session")
def gpu():
    if not _has_gpu():
        pytest.fail("GPU test requires a CUDA device (run under gpurun)")
    return 0
