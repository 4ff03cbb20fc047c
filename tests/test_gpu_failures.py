"""Device failures surface the way the reference's failing bodies do (-m gpu).

Reference engine.py:154-157, 227-243: a body that raises poisons the engine;
``wait_all`` raises EngineFailedError whose ``__cause__`` is the original
exception, the first failure wins and the engine stays poisoned.  On the GPU
path the "body" is a kernel: DPOTRF reports a non-positive pivot through a
status word read back at completion (cause: NotPositiveDefiniteError, a
numpy.linalg.LinAlgError like the oracle's np.linalg.cholesky raises), and a
failing launch or a device fault is a CudaError cause.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2308_15964_b200 as sf

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _spd_with_bad_pivot(b, col):
    """An SPD-looking tile whose leading minor of order col+1 is not positive."""
    rng = np.random.default_rng(b + col)
    R = rng.random((b, b)) * 0.01
    A = (R + R.T) / 2 + b * np.eye(b) * 0.01 + np.eye(b)
    A[col, col] = -1.0
    return A


@pytest.mark.parametrize("b,col,op", [(256, 5, "potrf"), (256, 100, "potrf_inv"), (256, 200, "potrf_fullinv"),
                                      (100, 70, "potrf"), (1024, 777, "potrf_fullinv")])
def test_non_spd_tile_poisons_engine_with_linalg_cause(b, col, op):
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 4), device_memory=1 << 30)
    try:
        A = _spd_with_bad_pivot(b, col)
        g = sf.TaskGraph().compute_on(eng)
        g.task(sf.write(A), device=getattr(sf.ops, op))
        with pytest.raises(sf.EngineFailedError) as ei:
            g.wait_all(timeout=60)
        cause = ei.value.__cause__
        assert isinstance(cause, sf.NotPositiveDefiniteError), repr(cause)
        assert isinstance(cause, np.linalg.LinAlgError)
        assert f"order {col + 1} " in str(cause), str(cause)
        # the engine stays poisoned: later work fails the same way (first failure wins)
        B = np.eye(64) * 2.0
        g2 = sf.TaskGraph().compute_on(eng)
        g2.task(sf.write(B), device=sf.ops.potrf)
        with pytest.raises(sf.EngineFailedError) as e2:
            g2.wait_all(timeout=60)
        assert f"order {col + 1} " in str(e2.value.__cause__)
    finally:
        eng.stop()


def test_spd_tiles_do_not_trip_the_status_word():
    """Thousands of POTRFs recycle the status slots; none reports a failure."""
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 4), device_memory=1 << 30)
    try:
        g = sf.TaskGraph().compute_on(eng)
        tiles = [np.eye(64) * 4.0 + 0.01 for _ in range(16)]
        for _ in range(300):
            for t in tiles:
                g.task(sf.write(t), device=sf.ops.dpotrf())
                g.task(sf.write(t), device=sf.ops.fill_spd(3, 0, 0, 64))
        assert g.wait_all(timeout=120)
    finally:
        eng.stop()


def test_failing_launch_poisons_engine_with_cuda_cause():
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 2), device_memory=1 << 28)
    try:
        c = sf.Cell(0)
        g = sf.TaskGraph().compute_on(eng)
        g.task(sf.write(c), device=sf.ops.cell("write", 1, 1))
        g.task(sf.write(c), device=sf.ops.fault("launch"))
        g.task(sf.write(c), device=sf.ops.cell("write", 1, 1))
        with pytest.raises(sf.EngineFailedError) as ei:
            g.wait_all(timeout=60)
        assert isinstance(ei.value.__cause__, sf.CudaError), repr(ei.value.__cause__)
        assert "invalid" in str(ei.value.__cause__).lower()
    finally:
        eng.stop()
    # the CUDA context survived the launch error: a fresh engine works
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 2), device_memory=1 << 28)
    try:
        c = sf.Cell(5)
        g = sf.TaskGraph().compute_on(eng)
        g.task(sf.write(c), device=sf.ops.add_i64(3))
        g.flush_to_host(c)
        assert g.wait_all(timeout=60) and c.value == 8
    finally:
        eng.stop()


def test_device_trap_poisons_engine_in_a_throwaway_process():
    code = r"""
import os, sys
sys.path.insert(0, %r)
import paper_2308_15964_b200 as sf
eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 2), device_memory=1 << 28)
c = sf.Cell(0)
g = sf.TaskGraph().compute_on(eng)
g.task(sf.write(c), device=sf.ops.fault("trap"))
try:
    g.wait_all(timeout=60)
    print("NO-ERROR", flush=True)
except sf.EngineFailedError as e:
    print("CAUGHT", type(e.__cause__).__name__, str(e.__cause__)[:200], flush=True)
os._exit(0)
""" % ROOT
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert "CAUGHT CudaError" in r.stdout, (r.stdout, r.stderr[-2000:])
