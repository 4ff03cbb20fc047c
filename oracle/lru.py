"""LRU models of a device arena.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* ``ReferenceLRU`` restates the reference's independent model
  (reference tests/test_device.py:37-54): a capacity counter and the victim
  order (stamp, hid).
* ``ArenaModel`` restates the reference arena itself (reference
  src/device.py:78-116 first-fit free list with coalescing, and
  src/device.py:208-264 LRU eviction by (stamp, hid) among unpinned blocks
  plus the fragmentation retry loop), with an allocation granularity.
"""

from __future__ import annotations


class ReferenceLRU:
    def __init__(self, capacity):
        self.capacity = capacity
        self.blocks = {}  # hid -> (size, stamp)
        self.clock = 0

    def access(self, hid, size):
        self.clock += 1
        if hid in self.blocks:
            self.blocks[hid] = (self.blocks[hid][0], self.clock)
            return
        used = sum(s for s, _ in self.blocks.values())
        while self.capacity - used < size:
            victim = min(self.blocks, key=lambda h: (self.blocks[h][1], h))
            used -= self.blocks.pop(victim)[0]
        self.blocks[hid] = (size, self.clock)


class StagingFailure(Exception):
    pass


class ArenaModel:
    def __init__(self, capacity, align=8):
        self.capacity = capacity
        self.align = align
        self.free = [(0, capacity)]
        self.blocks = {}  # hid -> [offset, size, stamp, pins]
        self.clock = 0
        self.evicted = []

    def _size(self, n):
        a = self.align
        return max((n + a - 1) // a * a, a)

    def _alloc(self, size):
        for i, (off, seg) in enumerate(self.free):
            if seg >= size:
                if seg == size:
                    del self.free[i]
                else:
                    self.free[i] = (off + size, seg - size)
                return off
        return None

    def _release(self, off, size):
        self.free.append((off, size))
        self.free.sort()
        merged = []
        for o, s in self.free:
            if merged and merged[-1][0] + merged[-1][1] == o:
                merged[-1] = (merged[-1][0], merged[-1][1] + s)
            else:
                merged.append((o, s))
        self.free = merged

    def free_bytes(self):
        return sum(s for _, s in self.free)

    def _victim(self):
        cands = [(b[2], h) for h, b in self.blocks.items() if b[3] == 0]
        if not cands:
            return None
        return min(cands)[1]

    def _evict(self, hid):
        off, size, _, _ = self.blocks.pop(hid)
        self._release(off, size)
        self.evicted.append(hid)

    def touch(self, hid, nbytes):
        """Stage hid (device.py:234-264) and stamp it (device.py:359)."""
        size = self._size(nbytes)
        if size > self.capacity:
            raise StagingFailure("oversize")
        if hid not in self.blocks:
            while self.free_bytes() < size:
                v = self._victim()
                if v is None:
                    raise StagingFailure("pinned")
                self._evict(v)
            off = self._alloc(size)
            while off is None:
                v = self._victim()
                if v is None:
                    raise StagingFailure("fragmentation")
                self._evict(v)
                off = self._alloc(size)
            self.blocks[hid] = [off, size, 0, 0]
        self.clock += 1
        self.blocks[hid][2] = self.clock
