"""Host buffers: pinned tile allocation and object -> (pointer, 2-D descriptor).

The reference moves objects through a three-method movable protocol or the
buffer tier (src/device.py:136-194).  The GPU engine replaces the Python
callbacks by a host pointer plus a descriptor registered once per handle
(sfx_register): rows, cols, ld and dtype.  Accepted objects:

* C-contiguous numpy arrays (float64 tiles; int64; anything else as bytes),
* writable contiguous buffers (bytearray, memoryview, array.array),
* :class:`~paper_2308_15964_b200.cell.Cell` (8-byte pinned scalar).

Objects that only implement ``move_to_device``/``move_from_device`` would need
Python callbacks on the copy path; they are refused at insertion with a
ConfigurationError rather than failing during staging.
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _native as N
from .errors import ConfigurationError

_finalizers = {}


def pinned_empty(shape, dtype=np.float64, sim: bool = False) -> np.ndarray:
    """numpy array backed by page-locked host memory (cudaHostAlloc).

    Pinned buffers make H2D/D2H copies truly asynchronous and run at full
    PCIe bandwidth; pageable buffers work too but copy through the driver's
    bounce buffer.
    """
    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dtype.itemsize
    ptr = ctypes.c_void_p()
    N.check(N.lib.sfx_host_alloc(max(nbytes, 1), 1 if sim else 0, ctypes.byref(ptr)))
    buf = (ctypes.c_char * max(nbytes, 1)).from_address(ptr.value)
    arr = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)
    addr = ptr.value
    weakref.finalize(buf, N.lib.sfx_host_free, ctypes.c_void_p(addr), 1 if sim else 0)
    return arr


def pinned_zeros(shape, dtype=np.float64, sim: bool = False) -> np.ndarray:
    a = pinned_empty(shape, dtype, sim)
    a[...] = 0
    return a


class HostDesc:
    __slots__ = ("ptr", "nbytes", "rows", "cols", "ld", "dtype", "keep")

    def __init__(self, ptr, nbytes, rows, cols, ld, dtype, keep):
        self.ptr = ptr
        self.nbytes = nbytes
        self.rows = rows
        self.cols = cols
        self.ld = ld
        self.dtype = dtype
        self.keep = keep


def describe(obj) -> HostDesc:
    """Host pointer and 2-D descriptor of a device-movable object."""
    sfx_buf = getattr(obj, "__sfx_buffer__", None)
    if sfx_buf is not None:
        obj = sfx_buf()
    if isinstance(obj, np.ndarray):
        if not obj.flags.c_contiguous or not obj.flags.writeable:
            raise ConfigurationError(
                "device operands must be writable C-contiguous arrays (reference device.py:189-193)")
        ptr = obj.ctypes.data
        if obj.dtype == np.float64 and obj.ndim in (1, 2):
            rows, cols = (obj.shape if obj.ndim == 2 else (1, obj.shape[0]))
            return HostDesc(ptr, obj.nbytes, rows, cols, cols, N.DTYPE_F64, obj)
        if obj.dtype == np.int64 and obj.ndim in (1, 2):
            rows, cols = (obj.shape if obj.ndim == 2 else (1, obj.shape[0]))
            return HostDesc(ptr, obj.nbytes, rows, cols, cols, N.DTYPE_I64, obj)
        return HostDesc(ptr, obj.nbytes, 1, obj.nbytes, obj.nbytes, N.DTYPE_BYTES, obj)
    try:
        view = memoryview(obj)
    except TypeError:
        raise ConfigurationError(
            f"{type(obj).__name__} is not device-movable on the GPU engine: pass a contiguous "
            "numpy array / writable buffer or a Cell") from None
    if view.readonly or not view.contiguous:
        raise ConfigurationError(
            f"{type(obj).__name__} exposes a buffer but it is not writable and contiguous")
    n = view.nbytes
    if n == 0:
        return HostDesc(0, 0, 1, 0, 0, N.DTYPE_BYTES, obj)
    cbuf = (ctypes.c_char * n).from_buffer(view.cast("B"))
    return HostDesc(ctypes.addressof(cbuf), n, 1, n, n, N.DTYPE_BYTES, (obj, cbuf))
