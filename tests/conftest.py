import os
import sys

import pytest

# Up to 8 ranks of the peer-memory path run as contexts of ONE process on the
# pool's single GPU, each on its own stream; their collectives spin-wait on the
# device.  With CUDA's default 8 hardware work queues two such streams can share
# a queue, and a spinning kernel then blocks the other rank's step behind it
# (a false dependency).  One process per GPU -- the real deployment -- never
# has this; the emulation needs more queues (set before CUDA initialises).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu():
    try:
        import ctypes
        cu = ctypes.CDLL("libcuda.so.1")
        if cu.cuInit(0) != 0:
            return False
        n = ctypes.c_int(0)
        return cu.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0
    except OSError:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
