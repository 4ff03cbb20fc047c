"""Registered device ops: what a ``device=`` argument names in the GPU engine.

In the reference a device task is a Python callable run on a simulated-device
worker thread with ``DeviceView`` arguments (src/engine.py:144-149).  On the
B200 path a device task names one of these ops instead; its operands are the
task's declared accesses in declaration order, exactly as the reference passes
views in declaration order (README.md:50-53).  Each op is a hand-written
sm_100a kernel sequence inside libsfx.so.

Operand conventions (tiles are 2-D row-major float64 arrays):

  dgemm(alpha, beta, trans_b)   A(r), B(r), C(w):  C = beta*C + alpha*A*op(B)
  gemm_nn                       C += A @ B            (tiled DGEMM configs)
  gemm_nt_sub                   C -= A @ B.T          (Cholesky trailing update)
  dsyrk(alpha, beta)            A(r), C(w): lower(C) = beta*C + alpha*A*A^T
  syrk_sub                      lower(C) -= A @ A.T
  dtrsm()                       L(r), B(w): B = B * L^-T  (right, lower, trans)
  dpotrf()                      A(w): lower(A) = chol(A) (upper untouched, LAPACK 'L')
  dpotrf(store_inverses=True)   + inv(L_jj)^T of each 64x64 diagonal block in its strict upper
  dtrsm(inverse_blocks=True)    B = B * L^-T using those blocks (DMMA GEMM sweeps)
  p2p_pair(eps2)                P_i(r), P_j(r), F_i(cw), F_j(cw)
  p2p_self(eps2)                P_i(r), F_i(cw)
  fill_uniform/fill_spd/fill_particles/zero   generators (write one tile)
  noop, spin(ns), cell(kind, a, b), bytes_add(off, length, delta)   runtime tests
"""

from __future__ import annotations

from . import _native as N


class Op:
    """An op code plus its scalar parameters (immutable)."""

    __slots__ = ("name", "code", "fparam", "iparam")

    def __init__(self, name, code, fparam=(0.0, 0.0, 0.0, 0.0), iparam=(0, 0, 0, 0)):
        self.name = name
        self.code = code
        self.fparam = tuple(float(x) for x in (list(fparam) + [0.0] * 4)[:4])
        self.iparam = tuple(int(x) for x in (list(iparam) + [0] * 4)[:4])

    def __repr__(self):
        return f"<op {self.name}>"

    def __eq__(self, other):
        return (isinstance(other, Op) and self.code == other.code and self.fparam == other.fparam
                and self.iparam == other.iparam)

    def __hash__(self):
        return hash((self.code, self.fparam, self.iparam))


def dgemm(alpha: float = 1.0, beta: float = 1.0, trans_b: bool = False) -> Op:
    return Op("dgemm", N.OP_DGEMM, (alpha, beta), (1 if trans_b else 0,))


def dsyrk(alpha: float = -1.0, beta: float = 1.0) -> Op:
    return Op("dsyrk", N.OP_DSYRK, (alpha, beta))


def dtrsm(inverse_blocks=False) -> Op:
    """B = B L^-T.  ``inverse_blocks=True``: L's tile comes from ``dpotrf(store_inverses=True)``
    and carries the inverses of its 64x64 diagonal blocks in its upper triangle, so the
    solve runs as DMMA GEMM sweeps (x inverse block, then trailing update).
    ``inverse_blocks="full"``: L's tile comes from ``dpotrf(store_inverses="full")`` and
    carries inv(L)^T in its strict upper triangle: the solve is ONE parallel DMMA GEMM."""
    if inverse_blocks == "full":
        return Op("dtrsm_fullinv", N.OP_DTRSM, iparam=(2,))
    return Op("dtrsm_inv" if inverse_blocks else "dtrsm", N.OP_DTRSM, iparam=(1 if inverse_blocks else 0,))


def dpotrf(store_inverses=False) -> Op:
    """Lower Cholesky in place.  Default: LAPACK 'L' semantics (upper triangle untouched).
    ``store_inverses=True``: the strict upper triangle of each 64x64 diagonal block receives
    inv(L_jj)^T (for ``dtrsm(inverse_blocks=True)``); ``"full"``: the whole strict upper
    triangle receives inv(L)^T (n = 64 * 2^k, 128 <= n <= 2048; for
    ``dtrsm(inverse_blocks="full")``).  The factor L is identical in every mode."""
    if store_inverses == "full":
        return Op("dpotrf_fullinv", N.OP_DPOTRF, iparam=(2,))
    return Op("dpotrf_inv" if store_inverses else "dpotrf", N.OP_DPOTRF, iparam=(1 if store_inverses else 0,))


def p2p_pair(eps2: float = 1e-9) -> Op:
    return Op("p2p_pair", N.OP_P2P_PAIR, (eps2,))


def p2p_self(eps2: float = 1e-9) -> Op:
    return Op("p2p_self", N.OP_P2P_SELF, (eps2,))


def fill_uniform(seed: int, row0: int, col0: int, ncols_total: int) -> Op:
    return Op("fill_uniform", N.OP_FILL_UNIFORM, iparam=(seed, row0, col0, ncols_total))


def fill_spd(seed: int, row0: int, col0: int, n: int) -> Op:
    return Op("fill_spd", N.OP_FILL_SPD, iparam=(seed, row0, col0, n))


def fill_particles(seed: int, first: int) -> Op:
    return Op("fill_particles", N.OP_FILL_PARTICLES, iparam=(seed, first))


def zero() -> Op:
    return Op("zero", N.OP_ZERO)


def dacc() -> Op:
    """A += B1 + ... + Bk (k <= 7): sums per-GPU partial accumulators into their target."""
    return Op("dacc", N.OP_DACC)


def spin(ns: int) -> Op:
    return Op("spin", N.OP_SPIN, iparam=(int(ns),))


def cell(kind: str, a: int = 1, b: int = 0) -> Op:
    """Cell arithmetic of the reference random programs (tests/conftest.py:87-124)."""
    kinds = {"read": 0, "write": 1, "maybe": 2, "atomic": 3, "commute": 4}
    return Op(f"cell_{kind}", N.OP_CELL, iparam=(kinds[kind], a, b))


def bytes_add(off: int, length: int, delta: int) -> Op:
    return Op("bytes_add", N.OP_BYTES_ADD, iparam=(off, length, delta))


def add_i64(delta: int) -> Op:
    """Every operand (an int64 cell) += delta with device atomics.  An op that
    accumulates atomically: its commutative_write members of one group run
    concurrently on one device (shared guard; the P2P ops behave the same)."""
    return Op("add_i64", N.OP_ADD_I64, iparam=(int(delta),))


def fault(kind: str = "launch") -> Op:
    """Failure injection (engine-failure tests): ``"launch"`` = a kernel launch with an
    invalid configuration (the launch fails; the CUDA context survives), ``"trap"`` = a
    device-side trap (sticky: the process's CUDA context is lost)."""
    return Op(f"fault_{kind}", N.OP_FAULT, iparam=({"launch": 0, "trap": 1}[kind],))


noop = Op("noop", N.OP_NOOP)
gemm_nn = dgemm(1.0, 1.0, False)
gemm_nt_sub = dgemm(-1.0, 1.0, True)
syrk_sub = dsyrk(-1.0, 1.0)
trsm = dtrsm()
potrf = dpotrf()
trsm_inv = dtrsm(inverse_blocks=True)
potrf_inv = dpotrf(store_inverses=True)
trsm_fullinv = dtrsm(inverse_blocks="full")
potrf_fullinv = dpotrf(store_inverses="full")


# -- user ops: the reference's device= callables (src/engine.py:144-149) ----------
#
# Two ways to run code of one's own on a task's staged operands:
#
#   * a NATIVE launcher (C ABI ``sfx_user_launch_fn`` in include/sfx.h, e.g.
#     examples/user_daxpy.cu) registered once with ``register(name, fn)``; the
#     executor thread calls it outside the runtime lock with the operands'
#     device pointers and the task's stream -- no Python, no GIL on the path;
#   * a PYTHON callable passed as ``device=`` exactly as in the reference:
#     ``graph.task(Read(x), Write(y), device=lambda vx, vy: ...)``.  It runs on
#     the device's executor thread with one ``DeviceView`` per access in
#     declaration order; with torch imported its work is enqueued on the task's
#     stream (``torch.cuda.ExternalStream``), so ``vy.array().add_(vx.array())``
#     runs in the task's place in the dependency order.  This puts the GIL on the
#     executor's path for those tasks only.
#
# A launcher returning non-zero (or a callable raising) fails the task: the
# engine is poisoned and ``wait_all`` raises EngineFailedError whose
# ``__cause__`` is the callable's exception (TaskFailedError for a native one),
# as in the reference (engine.py:154-157, 227-243).

import ctypes as _ct
import itertools as _it
import sys as _sys
import threading as _th

_DT = {N.DTYPE_F64: "float64", N.DTYPE_I64: "int64", N.DTYPE_BYTES: "uint8"}
_DT_SIZE = {N.DTYPE_F64: 8, N.DTYPE_I64: 8, N.DTYPE_BYTES: 1}
_registered = {}          # name -> (Op, keep-alive)
_reg_lock = _th.Lock()
_py_fns = {}              # key -> callable of a submitted, not yet executed task
_py_results = {}          # key -> non-None return value
_py_errors = []           # exceptions raised by callables (first failure wins)
_py_keys = _it.count(1)
_py_op = None


class DeviceView:
    """What a user op receives per access (reference src/device.py:119-133):
    ``device`` (runtime device index), ``size`` (bytes), ``descriptor``
    ((rows, cols, ld, dtype)), ``mode`` (access code), ``ptr`` (device address;
    host address on the simulated backend), ``stream`` (cudaStream_t as int,
    None on the simulated backend) and ``data`` (a writable memoryview of the
    block on the simulated backend, None on a GPU)."""

    __slots__ = ("device", "offset", "size", "descriptor", "data", "mode", "ptr", "stream")

    def __init__(self, v, stream):
        self.device = v.device
        self.offset = 0
        self.size = v.bytes
        self.descriptor = (v.rows, v.cols, v.ld, _DT.get(v.dtype, "uint8"))
        self.mode = v.mode
        self.ptr = v.data or 0
        self.stream = stream or None
        self.data = None
        if self.stream is None and self.ptr:
            self.data = memoryview((_ct.c_char * self.size).from_address(self.ptr)).cast("B")

    def __len__(self):
        return self.size

    @property
    def __cuda_array_interface__(self):
        if self.stream is None:
            raise AttributeError("simulated-backend views are host memory (use .data / .array())")
        rows, cols, ld, dt = self.descriptor
        item = {"float64": 8, "int64": 8}.get(dt, 1)
        return {"shape": (rows, cols), "typestr": {"float64": "<f8", "int64": "<i8"}.get(dt, "|u1"),
                "data": (self.ptr, False), "strides": (ld * item, item), "version": 3,
                "stream": None}  # the caller already runs on the task's stream

    def array(self):
        """The operand as a (rows, cols) array with row stride ld: a torch tensor
        sharing the device block on a GPU, a numpy array over the host block on the
        simulated backend."""
        if self.stream is None:
            import numpy as np
            rows, cols, ld, dt = self.descriptor
            item = np.dtype(dt).itemsize
            return np.ndarray((rows, cols), dtype=dt, buffer=self.data, strides=(ld * item, item))
        import torch
        return torch.as_tensor(self, device="cuda")

    def torch_stream(self):
        import torch
        return torch.cuda.ExternalStream(self.stream)


def _call_python(views, n, stream, fparam, iparam, user):
    key = iparam[0]
    fn = _py_fns.pop(key, None)
    try:
        if fn is None:
            raise RuntimeError(f"python device callable #{key} is not registered")
        vs = [DeviceView(views[k], stream) for k in range(n)]
        torch = _sys.modules.get("torch")
        if stream and torch is not None:
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                r = fn(*vs)
        else:
            r = fn(*vs)
        if r is not None:
            _py_results[key] = r
        return 0
    except BaseException as e:  # noqa: BLE001 -- the engine is poisoned with it (engine.py:154-157)
        _py_errors.append(e)
        return 1


def register(name: str, fn, fparam=(0.0, 0.0, 0.0, 0.0), iparam=(0, 0, 0, 0)) -> Op:
    """Register a user op under ``name`` and return its Op (``op.params(...)`` makes
    variants with other scalar parameters).  ``fn`` is a native launcher: a ctypes
    function pointer (e.g. ``ctypes.CDLL(path).sfx_example_daxpy``) or its address
    as an int; or a Python callable ``fn(*views) -> int`` with the launcher's
    signature wrapped for you (views as DeviceView, returns 0 on success)."""
    with _reg_lock:
        if name in _registered:
            raise ValueError(f"user op {name!r} is already registered")
        keep = None
        if isinstance(fn, int):
            addr = fn
        elif isinstance(fn, _ct._CFuncPtr) and not isinstance(fn, N.USER_LAUNCH):
            addr = _ct.cast(fn, _ct.c_void_p).value
            keep = fn
        elif isinstance(fn, N.USER_LAUNCH):
            addr, keep = _ct.cast(fn, _ct.c_void_p).value, fn
        elif callable(fn):
            def tramp(views, n, stream, fp, ip, user, _fn=fn):
                try:
                    return int(_fn(*[DeviceView(views[k], stream) for k in range(n)]) or 0)
                except BaseException as e:  # noqa: BLE001
                    _py_errors.append(e)
                    return 1
            keep = N.USER_LAUNCH(tramp)
            addr = _ct.cast(keep, _ct.c_void_p).value
        else:
            raise TypeError(f"register: need a launcher or a callable, got {fn!r}")
        code = _ct.c_uint32(0)
        N.check(N.lib.sfx_register_op(name.encode(), addr, None, _ct.byref(code)))
        op = Op(name, code.value, fparam, iparam)
        _registered[name] = (op, keep)
        return op


def _params(self, fparam=None, iparam=None) -> Op:
    return Op(self.name, self.code, self.fparam if fparam is None else fparam,
              self.iparam if iparam is None else iparam)


Op.params = _params


def python_callable(fn) -> Op:
    """The Op for one task whose body is the Python callable ``fn`` (graph.task
    does this for ``device=<callable>``)."""
    global _py_op
    if _py_op is None:
        with _reg_lock:
            if _py_op is None:
                keep = N.USER_LAUNCH(_call_python)
                code = _ct.c_uint32(0)
                N.check(N.lib.sfx_register_op(b"python_callable", _ct.cast(keep, _ct.c_void_p).value, None,
                                              _ct.byref(code)))
                _registered["python_callable"] = (Op("python_callable", code.value), keep)
                _py_op = code.value
    key = next(_py_keys)
    _py_fns[key] = fn
    return Op(getattr(fn, "__name__", "python_callable"), _py_op, iparam=(key,))


def take_error():
    """The first exception a user callable raised since the last call (or None)."""
    if not _py_errors:
        return None
    e = _py_errors[0]
    _py_errors.clear()
    return e


def result_of(op: Op):
    """The non-None value a Python callable task returned (KeyError if none)."""
    return _py_results.pop(op.iparam[0])
