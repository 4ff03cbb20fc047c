"""Restatement of the reference STF runtime for host worker threads.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the parity oracle for the
dependency trace / execution order, and the CPU baseline engine that
``bench.py`` times on the GPU box's host cores.

Reference sections restated here (paths relative to /root/reference/pkg/src/seqflow):

  access modes -> slot categories ........ access.py:16-51
  slot grouping (append_access) .......... handles.py:209-236
  pending counter + insertion guard ...... task.py:76, 105-124
  insertion, duplicate check, commute
  handles sorted by hid .................. graph.py:113-166
  commutative all-or-nothing guards ...... handles.py:249-270
  release / advance / commute re-offer ... handles.py:274-343
  FIFO and priority schedulers ........... scheduler.py:66-126
  worker loop and execute ................ engine.py:87-174
  trace events, successor edges .......... trace.py:27-102

Simplifications (not on the north-star path): no speculation, no
communication tasks, no device workers, no array views.  Bodies are plain
Python callables receiving the declared objects in declaration order.
"""

from __future__ import annotations

import heapq
import itertools
import threading
import time
from collections import deque

READ = "read"
WRITE = "write"
ATOMIC = "atomic_write"
COMMUTE = "commutative_write"
MAYBE = "maybe_write"
MODES = (READ, WRITE, ATOMIC, COMMUTE, MAYBE)

# access.py:41-47 -- READ/ATOMIC/COMMUTE group, WRITE/MAYBE are exclusive
CATEGORY = {READ: "R", ATOMIC: "A", COMMUTE: "C", WRITE: "X", MAYBE: "X"}

PUSH, POP, START, END = "Push", "Pop", "TaskStart", "TaskEnd"


class OracleError(Exception):
    pass


class _Slot:
    __slots__ = ("cat", "tasks", "done")

    def __init__(self, cat):
        self.cat = cat
        self.tasks = []
        self.done = 0


class _Handle:
    __slots__ = ("hid", "obj", "slots", "active", "lock", "guard")

    def __init__(self, hid, obj):
        self.hid = hid
        self.obj = obj
        self.slots = []
        self.active = 0
        self.lock = threading.Lock()
        self.guard = None


class _Task:
    __slots__ = ("index", "body", "priority", "name", "accesses", "objs", "pending",
                 "state", "queued", "lock", "commute", "held", "released", "result")

    def __init__(self, index, body, priority, name):
        self.index = index
        self.body = body
        self.priority = priority
        self.name = name
        self.accesses = []  # [handle, mode, slot_index]
        self.objs = []
        self.pending = 1  # insertion guard (task.py:76)
        self.state = "inserted"
        self.queued = False
        self.lock = threading.Lock()
        self.commute = []
        self.held = []
        self.released = False
        self.result = None

    def dec_pending(self):
        # task.py:109-124 (no disabled state without speculation)
        with self.lock:
            self.pending -= 1
            if self.pending > 0:
                return False
            if self.pending < 0:
                raise OracleError(f"negative pending on task {self.index}")
            self.state = "ready"
            return True


class _Fifo:
    """scheduler.py:66-94 -- pop order equals push order."""

    def __init__(self):
        self.q = deque()

    def push(self, task):
        self.q.append(task)

    def pop(self):
        return self.q.popleft() if self.q else None


class _Prio:
    """scheduler.py:97-126 -- key (-priority, push sequence)."""

    def __init__(self):
        self.h = []
        self.seq = itertools.count()

    def push(self, task):
        heapq.heappush(self.h, (-task.priority, next(self.seq), task))

    def pop(self):
        return heapq.heappop(self.h)[2] if self.h else None


class Oracle:
    """One task graph attached to a pool of ``workers`` host threads.

    ``paused=True`` holds every worker until :meth:`resume`, which is the
    reference's gated-insertion protocol (tests/conftest.py:184-203: a gate
    task occupies the only worker while the program is inserted).
    """

    def __init__(self, workers: int = 1, scheduler: str = "fifo", trace: bool = True,
                 paused: bool = False):
        if scheduler not in ("fifo", "prio"):
            raise OracleError(f"unknown scheduler {scheduler!r}")
        self._sched = _Fifo() if scheduler == "fifo" else _Prio()
        self._lock = threading.Condition(threading.Lock())  # scheduler + park (engine.py:186-190)
        self._done_cv = threading.Condition(threading.Lock())
        self._commute_lock = threading.Lock()
        self._handles = {}  # id(obj) -> handle
        self._handle_list = []
        self._tasks = []
        self._inserted = 0
        self._completed = 0
        self._failure = None
        self._paused = paused
        self._stopping = False
        self._trace = trace
        self._events = []
        self._ev_lock = threading.Lock()
        self._t0 = time.perf_counter_ns()
        self._workers = [threading.Thread(target=self._loop, args=(w,), daemon=True)
                         for w in range(workers)]
        for th in self._workers:
            th.start()

    # -- trace (trace.py:47-50) ---------------------------------------------
    def _record(self, kind, wid, task):
        if self._trace:
            with self._ev_lock:
                self._events.append((kind, time.perf_counter_ns() - self._t0, wid, task.index))

    # -- insertion (graph.py:113-166, handles.py:209-236) -----------------------
    def _handle(self, obj):
        h = self._handles.get(id(obj))
        if h is None:
            h = _Handle(len(self._handle_list), obj)
            self._handles[id(obj)] = h
            self._handle_list.append(h)
        return h

    def task(self, accesses, body=None, priority: int = 0, name=None) -> int:
        """Insert one task; ``accesses`` is a list of (mode, obj).  Returns its insertion index."""
        task = _Task(len(self._tasks), body, priority, name)
        seen = set()
        for mode, obj in accesses:
            if mode not in CATEGORY:
                raise OracleError(f"unknown access mode {mode!r}")
            h = self._handle(obj)
            if h.hid in seen:
                raise OracleError("task declares the same object twice")
            seen.add(h.hid)
            cat = CATEGORY[mode]
            with h.lock:
                slots = h.slots
                # join the last slot only if it groups, matches, and is not yet passed
                if cat != "X" and slots and slots[-1].cat == cat and h.active <= len(slots) - 1:
                    slot = slots[-1]
                else:
                    slot = _Slot(cat)
                    slots.append(slot)
                slot.tasks.append(task)
                index = len(slots) - 1
                if index != h.active:
                    with task.lock:
                        task.pending += 1
            task.accesses.append([h, mode, index])
            task.objs.append(obj)
        task.commute = sorted((a[0] for a in task.accesses if a[1] == COMMUTE), key=lambda h: h.hid)
        self._tasks.append(task)
        with self._done_cv:
            self._inserted += 1
        if task.dec_pending():
            self._push([task])
        return task.index

    # -- scheduling (engine.py:212-223) -----------------------------------------
    def _push(self, tasks, wid=-1):
        with self._lock:
            for t in tasks:
                with t.lock:
                    if t.queued:
                        continue
                    t.queued = True
                self._record(PUSH, wid, t)
                self._sched.push(t)
            self._lock.notify_all()

    def _loop(self, wid):
        while True:
            with self._lock:
                while True:
                    if self._stopping:
                        return
                    task = None
                    if not self._paused and self._failure is None:
                        task = self._sched.pop()
                    if task is not None:
                        with task.lock:
                            task.queued = False
                        break
                    self._lock.wait()
            self._execute(wid, task)

    # -- execution (engine.py:113-174) ------------------------------------------
    def _acquire(self, task):
        # handles.py:249-270
        if not task.commute:
            return True
        with self._commute_lock:
            taken = []
            for h in task.commute:
                if h.guard is None:
                    h.guard = task
                    taken.append(h)
                else:
                    for t in taken:
                        t.guard = None
                    return False
            task.held = taken
        return True

    def _execute(self, wid, task):
        self._record(POP, wid, task)
        with task.lock:
            if task.state != "ready":
                return
            task.state = "executing"
        if not self._acquire(task):
            with task.lock:
                task.state = "ready"
            self._push([task], wid)
            return
        self._record(START, wid, task)
        try:
            if task.body is not None:
                task.result = task.body(*task.objs)
        except BaseException as exc:  # fail-fast poisoning (engine.py:154-157)
            with self._done_cv:
                if self._failure is None:
                    self._failure = exc
                self._done_cv.notify_all()
            with self._lock:
                self._lock.notify_all()
            return
        self._record(END, wid, task)
        with task.lock:
            task.state = "finished"
        self._push(self._release(task), wid)

    # -- release (handles.py:274-343) -------------------------------------------
    def _release(self, task):
        ready = []
        with task.lock:
            if task.released:
                raise OracleError(f"double release of task {task.index}")
            task.released = True
        if task.held:
            with self._commute_lock:
                for h in task.held:
                    h.guard = None
            task.held = []
        touched = []
        for h, mode, index in task.accesses:
            with h.lock:
                slot = h.slots[index]
                slot.done += 1
                if index == h.active and slot.done >= len(slot.tasks):
                    h.active += 1
                    if h.active < len(h.slots):
                        for member in h.slots[h.active].tasks:
                            if member.dec_pending():
                                ready.append(member)
            if mode == COMMUTE:
                touched.append(h)
        for h in touched:  # re-offer commute members that lost a guard race
            with h.lock:
                if h.active >= len(h.slots) or h.slots[h.active].cat != "C":
                    continue
                for other in h.slots[h.active].tasks:
                    if other is not task:
                        with other.lock:
                            if other.state == "ready" and not other.queued:
                                ready.append(other)
        with self._done_cv:
            self._completed += 1
            self._done_cv.notify_all()
        return ready

    # -- control ----------------------------------------------------------------
    def resume(self):
        with self._lock:
            self._paused = False
            self._lock.notify_all()

    def wait_all(self, timeout=None) -> bool:
        deadline = None if timeout is None else time.monotonic() + timeout
        with self._done_cv:
            while True:
                if self._failure is not None:
                    raise OracleError("a task body failed") from self._failure
                if self._completed >= self._inserted:
                    return True
                if deadline is not None and time.monotonic() >= deadline:
                    return False
                self._done_cv.wait(timeout=0.5)

    def stop(self):
        with self._lock:
            self._stopping = True
            self._lock.notify_all()
        for th in self._workers:
            th.join()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.stop()
        return False

    # -- exports ------------------------------------------------------------------
    def edges(self) -> set:
        """Successor pairs (src, dst) as insertion indices (trace.py:94-102)."""
        out = set()
        for h in self._handle_list:
            for a, b in zip(h.slots, h.slots[1:]):
                for s in a.tasks:
                    for d in b.tasks:
                        out.add((s.index, d.index))
        return out

    def slot_layout(self) -> list:
        """Per handle (first-use order): [(category, [insertion indices])]."""
        return [[(s.cat, [t.index for t in s.tasks]) for s in h.slots] for h in self._handle_list]

    def events(self) -> list:
        with self._ev_lock:
            return sorted(self._events, key=lambda e: e[1])

    def pop_order(self) -> list:
        return [e[3] for e in self.events() if e[0] == POP]

    def start_order(self) -> list:
        return [e[3] for e in self.events() if e[0] == START]

    def results(self) -> list:
        return [t.result for t in self._tasks]


def static_successor_edges(programs_accesses) -> set:
    """Expected successor edges from first principles (reference tests/conftest.py:160-181).

    ``programs_accesses`` is a list (in insertion order) of lists of
    (mode, key) pairs; keys identify objects.  Per key, consecutive accesses of
    the same grouping category share a group (exclusive never groups); every
    member of a group links to every member of the next.
    """
    groups = {}
    for idx, accesses in enumerate(programs_accesses):
        for mode, key in accesses:
            cat = CATEGORY[mode]
            gl = groups.setdefault(key, [])
            if gl and gl[-1][0] == cat and cat != "X":
                gl[-1][1].append(idx)
            else:
                gl.append((cat, [idx]))
    edges = set()
    for gl in groups.values():
        for (_, src), (_, dst) in zip(gl, gl[1:]):
            edges.update((i, j) for i in src for j in dst)
    return edges
