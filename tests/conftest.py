"""Shared test configuration.

Markers: ``gpu`` -- needs a CUDA device (run on the B200 box with ``-m gpu``);
everything else runs on CPU (``-m "not gpu"``), using the simulated backend
for the native runtime's bookkeeping and the oracle for semantics.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"
REFERENCE_TESTS = "/root/reference/pkg/tests"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: longer-running test")


def reference_available() -> bool:
    return os.path.isdir(REFERENCE_SRC)


@pytest.fixture
def sim_engine():
    import paper_2308_15964_b200 as sf

    eng = sf.create_engine(sf.WorkerTeam.of_host_and_device_workers(devices=1, host_workers=1), backend="sim")
    yield eng
    eng.stop()


@pytest.fixture
def gpu_engine():
    import paper_2308_15964_b200 as sf

    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 4), device_memory=8 << 30)
    yield eng
    eng.stop()
