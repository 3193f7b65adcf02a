import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs libfpg.so kernels)")
    config.addinivalue_line("markers", "slow: long-running")


def gpu_available() -> bool:
    try:
        from paper_1711_08475_b200._lib import load_fpg
        import ctypes
        n = ctypes.c_int(0)
        return load_fpg().fpg_device_count(ctypes.byref(n)) == 0 and n.value > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built (reference tree absent when building)")
    return Reference()
