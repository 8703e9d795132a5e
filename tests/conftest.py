import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running parity case")


def gpu_available() -> bool:
    try:
        import ctypes
        from paper_2602_02204_b200 import dev_lib
        n = ctypes.c_int32()
        return dev_lib().omni_device_count(ctypes.byref(n)) == 0 and n.value > 0
    except Exception:
        return False
