import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device) to run")


def _has_gpu():
    try:
        import ctypes
        cudart = None
        for name in ("libcudart.so.12", "libcudart.so"):
            try:
                cudart = ctypes.CDLL(name)
                break
            except OSError:
                continue
        if cudart is None:
            return False
        n = ctypes.c_int(0)
        return cudart.cudaGetDeviceCount(ctypes.byref(n)) == 0 and n.value > 0
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def ref():
    from oracle import Oracle, available
    if not available("ref"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Oracle("ref")


@pytest.fixture(scope="session")
def port():
    from oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session", params=["ref", "port"])
def oracle_impl(request):
    from oracle import Oracle, available
    if not available(request.param):
        pytest.skip(f"oracle {request.param} not built")
    return Oracle(request.param)
