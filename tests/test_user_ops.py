"""User ops: the reference's ``device=`` callables (src/engine.py:144-149) on the
native runtime -- native launchers registered through ``sfx_register_op`` and
Python callables receiving DeviceViews (src/device.py:119-133).

The CPU tests run on the simulated backend (views are host memory, the
launcher computes synchronously); the ``gpu`` tests run the same programs on a
B200, with the native example launcher (examples/user_daxpy.cu) enqueueing its
kernel on the task's stream and torch work of a Python callable enqueued there
too.  Failure semantics follow the reference's test_engine.py: a failing body
poisons the engine and ``wait_all`` raises EngineFailedError with the body's
exception as ``__cause__``.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import pytest

import paper_2308_15964_b200 as sf
from paper_2308_15964_b200 import ops

PKG = os.path.dirname(sf.__file__)
_lib = None


def example_lib():
    global _lib
    if _lib is None:
        path = os.path.join(PKG, "libsfx_user_daxpy.so")
        if not os.path.exists(path):  # built by __graft_entry__.build(); build it if a checkout lacks it
            from paper_2308_15964_b200 import build as B
            B._build_examples(B._nvcc(), False, False)
        _lib = ctypes.CDLL(path)
    return _lib


_daxpy = None


def daxpy_op():
    global _daxpy
    if _daxpy is None:
        _daxpy = ops.register("example_daxpy", example_lib().sfx_example_daxpy)
    return _daxpy


def engine(backend, devices=1, streams=2):
    return sf.create_engine(sf.WorkerTeam.of_devices(devices, streams), backend=backend)


def _chain_program(g, xs, y, alpha_op):
    """y += 2 x0, then y += 2 x1, ... in one write chain on y."""
    for x in xs:
        g.task(sf.read(x), sf.write(y), device=alpha_op)


def _add_into(va, vb):
    B = vb.array()
    B += va.array()


def _scale(f):
    def body(v):
        X = v.array()
        X *= f
    return body


def run_native_daxpy(backend):
    op = daxpy_op().params(fparam=(2.0,))
    rng = np.random.default_rng(3)
    xs = [rng.standard_normal((48, 40)) for _ in range(5)]
    y = rng.standard_normal((48, 40))
    y0 = y.copy()
    eng = engine(backend)
    try:
        g = sf.TaskGraph().compute_on(eng)
        _chain_program(g, xs, y, op)
        g.flush_to_host(y)
        assert g.wait_all(timeout=60)
    finally:
        eng.stop()
    want = y0 + 2.0 * sum(xs)
    assert np.allclose(y, want, rtol=1e-14, atol=1e-14)


def run_python_callable(backend):
    rng = np.random.default_rng(5)
    a = rng.standard_normal((32, 32))
    b = np.zeros((32, 32))
    seen = []

    def body(va, vb):
        seen.append((va.descriptor, va.mode, vb.mode))
        A, B = va.array(), vb.array()
        B += 3.0 * A  # numpy (sim) or torch on the task's stream (GPU)
        return "done"

    eng = engine(backend)
    try:
        g = sf.TaskGraph().compute_on(eng)
        t1 = g.task(sf.read(a), sf.write(b), device=body)
        t2 = g.task(sf.read(a), sf.write(b), device=_add_into)
        g.flush_to_host(b)
        assert g.wait_all(timeout=60)
        assert t1.get_value() == "done" and t1.get_value() == "done"
        with pytest.raises(ValueError):
            t2.get_value()  # returned None: no value (task.py:260-261)
    finally:
        eng.stop()
    assert np.allclose(b, 4.0 * a, rtol=1e-15, atol=0)
    assert seen == [((32, 32, 32, "float64"), sf._native.READ, sf._native.WRITE)]


def run_failure(backend):
    class Boom(Exception):
        pass

    def bad(v):
        raise Boom("user body failed")

    x = np.zeros((8, 8))
    eng = engine(backend)
    try:
        g = sf.TaskGraph().compute_on(eng)
        g.task(sf.write(x), device=bad)
        with pytest.raises(sf.EngineFailedError) as ei:
            g.wait_all(timeout=60)
        assert isinstance(ei.value.__cause__, Boom)
    finally:
        eng.stop()


def run_native_failure(backend):
    # the example launcher rejects mismatched shapes: returns 1 -> TaskFailedError cause
    op = daxpy_op().params(fparam=(1.0,))
    x, y = np.zeros((8, 8)), np.zeros((4, 8))
    eng = engine(backend)
    try:
        g = sf.TaskGraph().compute_on(eng)
        g.task(sf.read(x), sf.write(y), device=op)
        with pytest.raises(sf.EngineFailedError) as ei:
            g.wait_all(timeout=60)
        assert isinstance(ei.value.__cause__, sf.errors.TaskFailedError)
        assert "example_daxpy" in str(ei.value)
    finally:
        eng.stop()


# -- CPU (simulated backend) ---------------------------------------------------

def test_registration_rules():
    daxpy_op()
    with pytest.raises(ValueError):
        ops.register("example_daxpy", example_lib().sfx_example_daxpy)
    code = ctypes.c_uint32(0)
    assert sf._native.lib.sfx_register_op(b"", None, None, ctypes.byref(code)) == sf._native.ERR_CONFIG
    assert daxpy_op().code >= sf._native.OP_USER_BASE


def test_native_launcher_on_sim():
    run_native_daxpy("sim")


def test_python_callable_on_sim():
    run_python_callable("sim")


def test_python_callable_failure_poisons_on_sim():
    run_failure("sim")


def test_native_launcher_failure_on_sim():
    run_native_failure("sim")


def test_user_ops_keep_dependency_order_on_sim():
    # a read of y between two writes sees exactly the first write (slot order)
    y = np.ones((4, 4))
    snaps = []
    eng = engine("sim", streams=4)
    try:
        g = sf.TaskGraph().compute_on(eng)
        for k in range(20):
            g.task(sf.write(y), device=_scale(2.0))
            g.task(sf.read(y), device=lambda v: snaps.append(float(v.array()[0, 0])))
        g.flush_to_host(y)
        assert g.wait_all(timeout=60)
    finally:
        eng.stop()
    assert snaps == [2.0 ** (k + 1) for k in range(20)]
    assert y[0, 0] == 2.0 ** 20


# -- GPU -----------------------------------------------------------------------

@pytest.mark.gpu
def test_native_launcher_on_gpu():
    run_native_daxpy("cuda")


@pytest.mark.gpu
def test_python_callable_with_torch_on_gpu():
    import torch  # noqa: F401  (callables' torch work goes on the task's stream)
    run_python_callable("cuda")


@pytest.mark.gpu
def test_user_ops_between_builtin_ops_on_gpu():
    """A native user op between two DMMA GEMMs on the same tile: C = A B; C += 2 X;
    C += A B -- ordering through CUDA events across streams."""
    import torch  # noqa: F401
    rng = np.random.default_rng(11)
    n = 256
    A, B, X = (rng.standard_normal((n, n)) for _ in range(3))
    C = np.zeros((n, n))
    op = daxpy_op().params(fparam=(2.0,))
    eng = engine("cuda", streams=4)
    try:
        g = sf.TaskGraph().compute_on(eng)
        g.task(sf.read(A), sf.read(B), sf.write(C), device=sf.ops.gemm_nn)
        g.task(sf.read(X), sf.write(C), device=op)
        g.task(sf.read(A), sf.read(B), sf.write(C), device=sf.ops.gemm_nn)
        g.task(sf.write(C), device=_scale(0.5))
        g.flush_to_host(C)
        assert g.wait_all(timeout=60)
    finally:
        eng.stop()
    want = 0.5 * (2 * (A @ B) + 2 * X)
    assert np.max(np.abs(C - want)) / np.max(np.abs(want)) < 1e-12


@pytest.mark.gpu
def test_python_callable_failure_poisons_on_gpu():
    run_failure("cuda")


@pytest.mark.gpu
def test_native_launcher_failure_on_gpu():
    run_native_failure("cuda")
