"""ctypes binding of libsfx.so (include/sfx.h).

The product path always goes through this library.  If it is missing the
import fails loudly: there is no Python or CPU fallback for device tasks.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import (
    ConfigurationError,
    DuplicateAccessError,
    EngineFailedError,
    InternalConsistencyError,
    RegistrationError,
    SeqflowError,
    StagingError,
    TaskFailedError,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsfx.so")

OK = 0
TIMEOUT = 1
ERR_CONFIG = -2
ERR_STAGING = -3
ERR_ENGINE_FAILED = -4
ERR_CUDA = -5
ERR_INTERNAL = -6
ERR_DUPLICATE = -7
ERR_REGISTRATION = -8
ERR_UNSUPPORTED = -9
ERR_NUMERIC = -10
ERR_USER = -11

READ, WRITE, ATOMIC_WRITE, COMMUTATIVE_WRITE, MAYBE_WRITE = 0, 1, 2, 3, 4

FLAG_SIM = 1
FLAG_TRACE = 2
FLAG_PAUSED = 4
FLAG_KTIME = 8

SCHED_FIFO, SCHED_PRIO = 0, 1

DTYPE_BYTES, DTYPE_F64, DTYPE_I64 = 0, 1, 2

OP_NOOP = 0
OP_SPIN = 1
OP_CELL = 2
OP_BYTES_ADD = 3
OP_FLUSH = 4
OP_EXTERN = 6
OP_FAULT = 7
OP_ADD_I64 = 5
OP_DGEMM = 10
OP_DSYRK = 11
OP_DTRSM = 12
OP_DPOTRF = 13
OP_P2P_PAIR = 20
OP_P2P_SELF = 21
OP_FILL_UNIFORM = 30
OP_FILL_SPD = 31
OP_FILL_PARTICLES = 32
OP_ZERO = 33
OP_DACC = 34
OP_USER_BASE, OP_USER_MAX = 256, 64  # sfx_register_op codes

EV_PUSH, EV_POP, EV_START, EV_END, EV_STAGE_BEGIN, EV_STAGE_END = range(6)
EV_NAMES = {EV_PUSH: "Push", EV_POP: "Pop", EV_START: "TaskStart", EV_END: "TaskEnd",
            EV_STAGE_BEGIN: "StageInBegin", EV_STAGE_END: "StageInEnd"}


class TaskDesc(ctypes.Structure):
    _fields_ = [
        ("tid", ctypes.c_uint64),
        ("graph", ctypes.c_uint32),
        ("op", ctypes.c_uint32),
        ("priority", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("n_access", ctypes.c_uint32),
        ("flags", ctypes.c_uint32),
        ("fparam", ctypes.c_double * 4),
        ("iparam", ctypes.c_int64 * 4),
    ]


class AccessDesc(ctypes.Structure):
    _fields_ = [("hid", ctypes.c_uint64), ("mode", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class DevStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "bytes_to_device", "copies_to_device", "bytes_from_device", "copies_from_device",
        "bytes_p2p_in", "copies_p2p_in", "hits", "misses", "evictions", "writebacks",
        "blocks", "bytes_in_use", "capacity", "tasks_executed", "kernel_launches", "stream_waits",
        "t_plan_ns", "t_issue_ns", "t_release_ns", "t_complete_ns", "groups", "prefetches",
        "timed_groups", "timed_tasks", "timed_ns", "busy_ns")] + [
        ("first_start_ns", ctypes.c_int64), ("last_end_ns", ctypes.c_int64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class Event(ctypes.Structure):
    _fields_ = [("t_ns", ctypes.c_int64), ("tid", ctypes.c_uint64), ("kind", ctypes.c_int32),
                ("worker", ctypes.c_int32), ("extra", ctypes.c_int64)]


class View(ctypes.Structure):
    """sfx_view: one staged operand handed to a user op's launcher."""
    _fields_ = [("data", ctypes.c_void_p), ("bytes", ctypes.c_uint64), ("rows", ctypes.c_int64),
                ("cols", ctypes.c_int64), ("ld", ctypes.c_int64), ("dtype", ctypes.c_int32),
                ("mode", ctypes.c_uint32), ("device", ctypes.c_int32), ("reserved", ctypes.c_int32)]


# int (*)(const sfx_view*, int, void* stream, const double* fparam, const int64_t* iparam, void* user)
USER_LAUNCH = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(View), ctypes.c_int, ctypes.c_void_p,
                               ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2308_15964_b200.build` "
            "(the GPU execution path has no Python fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    u32, u64, i32, i64, dbl = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "sfx_abi_version": ([], ctypes.c_int),
        "sfx_device_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
        "sfx_create": ([ctypes.c_int, P, ctypes.c_int, P, u32, u32, u32, ctypes.POINTER(P)], ctypes.c_int),
        "sfx_destroy": ([P], ctypes.c_int),
        "sfx_last_error": ([P], ctypes.c_char_p),
        "sfx_failure": ([P, ctypes.POINTER(ctypes.c_int), ctypes.c_char_p, u64], ctypes.c_int),
        "sfx_graph_create": ([P, ctypes.POINTER(u32)], ctypes.c_int),
        "sfx_register": ([P, u32, u64, P, u64, i64, i64, i64, i32], ctypes.c_int),
        "sfx_set_home": ([P, u64, i32], ctypes.c_int),
        "sfx_unregister": ([P, u64], ctypes.c_int),
        "sfx_submit": ([P, u32, P, P], ctypes.c_int),
        "sfx_pause": ([P], ctypes.c_int),
        "sfx_resume": ([P], ctypes.c_int),
        "sfx_wait_all": ([P, u32, dbl], ctypes.c_int),
        "sfx_wait_task": ([P, u64, dbl], ctypes.c_int),
        "sfx_task_state": ([P, u64, ctypes.POINTER(i32)], ctypes.c_int),
        "sfx_flush": ([P, u32, u64, u64, i32], ctypes.c_int),
        "sfx_stats": ([P, ctypes.c_int, ctypes.POINTER(DevStats)], ctypes.c_int),
        "sfx_resident": ([P, ctypes.c_int, P, u64, ctypes.POINTER(u64)], ctypes.c_int),
        "sfx_block_state": ([P, u64, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)], ctypes.c_int),
        "sfx_trace": ([P, u32, P, u64, ctypes.POINTER(u64)], ctypes.c_int),
        "sfx_edges": ([P, u32, P, P, P, u64, ctypes.POINTER(u64)], ctypes.c_int),
        "sfx_violations": ([P, ctypes.POINTER(u64)], ctypes.c_int),
        "sfx_set_option": ([P, ctypes.c_char_p, i64], ctypes.c_int),
        "sfx_host_alloc": ([u64, ctypes.c_int, ctypes.POINTER(P)], ctypes.c_int),
        "sfx_host_free": ([P, ctypes.c_int], ctypes.c_int),
        "sfx_fp64_peak": ([ctypes.c_int, ctypes.POINTER(dbl), ctypes.POINTER(dbl)], ctypes.c_int),
        "sfx_fp64_dfma_peak": ([ctypes.c_int, ctypes.POINTER(dbl)], ctypes.c_int),
        "sfx_extern_poll": ([P, ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64), ctypes.c_double],
                            ctypes.c_int),
        "sfx_extern_done": ([P, ctypes.c_uint64, ctypes.c_int, ctypes.c_char_p], ctypes.c_int),
        "sfx_gemm_paths": ([P, u32], ctypes.c_int),
        "sfx_fail": ([P, ctypes.c_char_p], ctypes.c_int),
        "sfx_graph_option": ([P, u32, ctypes.c_char_p, i64], ctypes.c_int),
        "sfx_live": ([P, ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(u64)], ctypes.c_int),
        "sfx_register_op": ([ctypes.c_char_p, P, P, ctypes.POINTER(u32)], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.sfx_abi_version() != 1:
        raise ImportError("libsfx.so ABI version mismatch; rebuild it")
    return lib


lib = _load()
EXPORTED = ("sfx_abi_version", "sfx_device_count", "sfx_create", "sfx_destroy", "sfx_last_error",
            "sfx_failure", "sfx_graph_create", "sfx_register", "sfx_set_home", "sfx_unregister",
            "sfx_submit", "sfx_pause", "sfx_resume", "sfx_wait_all", "sfx_wait_task",
            "sfx_task_state", "sfx_flush", "sfx_stats", "sfx_resident", "sfx_block_state",
            "sfx_trace", "sfx_edges", "sfx_violations", "sfx_set_option", "sfx_host_alloc", "sfx_host_free",
            "sfx_fp64_peak", "sfx_fp64_dfma_peak", "sfx_extern_poll", "sfx_extern_done", "sfx_gemm_paths", "sfx_fail",
            "sfx_graph_option", "sfx_live", "sfx_register_op")

GEMM_PATH_NAMES = ("launches", "tasks", "work_items", "cpref", "multi_tile", "cpref_multi_tile", "splitk", "tri",
                   "lower", "nn", "nt")


def gemm_paths() -> dict:
    """Process-wide DGEMM launch-path counters (sfx_gemm_paths)."""
    buf = (ctypes.c_uint64 * len(GEMM_PATH_NAMES))()
    lib.sfx_gemm_paths(buf, len(GEMM_PATH_NAMES))
    return dict(zip(GEMM_PATH_NAMES, list(buf)))

_ERRORS = {
    ERR_CONFIG: ConfigurationError,
    ERR_STAGING: StagingError,
    ERR_DUPLICATE: DuplicateAccessError,
    ERR_REGISTRATION: RegistrationError,
    ERR_INTERNAL: InternalConsistencyError,
    ERR_ENGINE_FAILED: EngineFailedError,
    ERR_UNSUPPORTED: ConfigurationError,
}


class CudaError(SeqflowError):
    """A CUDA runtime error (launch failure, fault) inside the GPU engine."""


_ERRORS[ERR_CUDA] = CudaError


class NotPositiveDefiniteError(SeqflowError, np.linalg.LinAlgError):
    """A DPOTRF tile had a non-positive leading minor (LAPACK info > 0).

    Also a ``numpy.linalg.LinAlgError``: the oracle's body (np.linalg.cholesky)
    raises that class, so the ``__cause__`` of the EngineFailedError has the same
    type on both paths (reference engine.py:154-157, 227-243)."""


_ERRORS[ERR_NUMERIC] = NotPositiveDefiniteError
_ERRORS[ERR_USER] = TaskFailedError  # a user op's launcher failed (a callable's own exception when it raised)


def error_for(code: int, msg: str) -> Exception:
    return _ERRORS.get(code, SeqflowError)(msg)


def check(rc: int, handle=None) -> int:
    if rc < 0:
        msg = lib.sfx_last_error(handle)
        raise error_for(rc, (msg or b"").decode(errors="replace"))
    return rc


def device_count() -> int:
    n = ctypes.c_int(0)
    lib.sfx_device_count(ctypes.byref(n))
    return n.value
