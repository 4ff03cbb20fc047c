"""Cell: a mutable scalar that can live on a device (reference src/cell.py:23-63).

The reference Cell packs its value with struct into the arena through the
movable protocol.  Here the value lives in an 8-byte host buffer that the
runtime stages directly (int64 for int/bool, float64 for float), so device
ops (e.g. the cell arithmetic of the reference random programs) read and
write it in place.  The 8-byte buffers are carved from page-locked slabs when
a GPU is present: copies of pageable memory go through the driver's staging
path, which under heavy eviction traffic stalled streams.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

_SLAB_SLOTS = 4096  # 8-byte cells per page-locked slab (32 KiB)
_slab = None
_slab_next = _SLAB_SLOTS
_slab_lock = threading.Lock()
_pinned_ok = None


def _cell_buffer(dtype) -> np.ndarray:
    """One 8-byte buffer: a slot of a pinned slab, or plain numpy without a GPU."""
    global _slab, _slab_next, _pinned_ok
    if _pinned_ok is False:
        return np.zeros(1, dtype=dtype)
    with _slab_lock:
        if _slab_next >= _SLAB_SLOTS:
            if _pinned_ok is None:
                from . import _native as N

                n = ctypes.c_int(0)
                _pinned_ok = N.lib.sfx_device_count(ctypes.byref(n)) == 0 and n.value > 0
                if not _pinned_ok:
                    return np.zeros(1, dtype=dtype)
            from .memory import pinned_empty

            _slab = pinned_empty((_SLAB_SLOTS,), np.int64)  # slabs live for the process
            _slab_next = 0
        buf = _slab[_slab_next:_slab_next + 1].view(dtype)
        _slab_next += 1
    buf[0] = 0
    return buf


def _kind(value):
    if type(value) is bool:
        return bool
    if type(value) is int:
        return int
    if type(value) is float:
        return float
    raise TypeError(f"Cell holds int, float, or bool, not {type(value).__name__}")


class Cell:
    __slots__ = ("_buf", "_kind", "__weakref__")

    def __init__(self, value=0):
        k = _kind(value)
        self._kind = k
        self._buf = _cell_buffer(np.float64 if k is float else np.int64)
        self.value = value

    @property
    def value(self):
        v = self._buf[0]
        if self._kind is bool:
            return bool(v)
        return float(v) if self._kind is float else int(v)

    @value.setter
    def value(self, v):
        k = _kind(v)
        if (k is float) != (self._kind is float):
            # the buffer is registered with the runtime by address: its dtype is fixed
            raise TypeError(f"this Cell stores {self._kind.__name__}; cannot assign {k.__name__}")
        self._kind = k
        self._buf[0] = v

    def __sfx_buffer__(self):
        return self._buf

    def __repr__(self):
        return f"Cell({self.value!r})"

    def __eq__(self, other):
        if isinstance(other, Cell):
            return self.value == other.value and type(self.value) is type(other.value)
        return NotImplemented

    def __hash__(self):
        return hash((type(self.value), self.value))

    def duplicate(self) -> "Cell":
        return Cell(self.value)

    def assign_from(self, other: "Cell") -> None:
        self.value = other.value
