"""Cell: a mutable scalar that can live on a device (reference src/cell.py:23-63).

The reference Cell packs its value with struct into the arena through the
movable protocol.  Here the value lives in an 8-byte host buffer that the
runtime stages directly (int64 for int/bool, float64 for float), so device
ops (e.g. the cell arithmetic of the reference random programs) read and
write it in place.
"""

from __future__ import annotations

import numpy as np


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
        self._buf = np.zeros(1, dtype=np.float64 if k is float else np.int64)
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
