"""Task graphs on the GPU engine (drop-in for reference src/graph.py:26-295).

Insertion keeps the reference's contract: one inserter thread, accesses in
declaration order, ``DuplicateAccessError`` for an object declared twice,
process-global task ids (task.py:63-69) and handle ids (handles.py:123-126),
``wait_all`` returning False on timeout and raising ``EngineFailedError``
(with the original error as ``__cause__``) after a failure.  Everything past
the access list -- slot binding, readiness, placement, staging, launch and
release -- happens in libsfx.so; Python never runs on the execution path.
"""

from __future__ import annotations

import contextlib
import ctypes
import enum
import itertools
import struct
import threading
import time

import numpy as np

from . import _native as N

try:  # CPython fast path for single-task submits (csrc/pyext/sfxfast.c); ctypes otherwise
    from . import _sfxfast
    _fast_submit1 = _sfxfast.submit1
    _fast_task = _sfxfast.task
except ImportError:  # pragma: no cover - the build makes it next to libsfx.so
    _sfxfast = _fast_submit1 = _fast_task = None
from . import memory
from . import ops as ops_mod
from .access import _CODES as _MODE_CODE
from .access import AccessMode, AccessSpec

if _sfxfast is not None:
    _sfxfast.bind_types(AccessSpec, ops_mod.Op)
from .errors import (
    ConfigurationError,
    DuplicateAccessError,
    EngineFailedError,
    RegistrationError,
    SpeculationError,
)

_tid_counter = itertools.count(1)
_hid_counter = itertools.count(1)
_id_lock = threading.Lock()


def _next_tid() -> int:
    if _sfxfast is not None:  # one process-global counter with the native fast path
        return _sfxfast.reserve_tids(1)
    with _id_lock:
        return next(_tid_counter)


def _reserve_tids(n: int) -> int:
    """First of ``n`` consecutive process-global task ids."""
    global _tid_counter
    if _sfxfast is not None:
        return _sfxfast.reserve_tids(n)
    with _id_lock:
        first = next(_tid_counter)
        _tid_counter = itertools.count(first + n)
    return first


def _next_hid() -> int:
    with _id_lock:
        return next(_hid_counter)


TASK_DTYPE = np.dtype({
    "names": ["tid", "graph", "op", "priority", "device", "n_access", "flags", "fparam", "iparam"],
    "formats": [np.uint64, np.uint32, np.uint32, np.int32, np.int32, np.uint32, np.uint32,
                (np.float64, 4), (np.int64, 4)],
    "offsets": [0, 8, 12, 16, 20, 24, 28, 32, 64],
    "itemsize": 96,
})
ACCESS_DTYPE = np.dtype({"names": ["hid", "mode", "reserved"], "formats": [np.uint64, np.uint32, np.uint32],
                         "offsets": [0, 8, 12], "itemsize": 16})
assert TASK_DTYPE.itemsize == ctypes.sizeof(N.TaskDesc)
_DESC = struct.Struct("<QIIiiII4d4q")
_ACC = struct.Struct("<QII")
assert _DESC.size == ctypes.sizeof(N.TaskDesc) and _ACC.size == ctypes.sizeof(N.AccessDesc)
assert ACCESS_DTYPE.itemsize == ctypes.sizeof(N.AccessDesc)


class TaskState(enum.Enum):
    INSERTED = "inserted"
    READY = "ready"
    EXECUTING = "executing"
    FINISHED = "finished"
    DISABLED = "disabled"


_STATE = {0: TaskState.INSERTED, 1: TaskState.READY, 2: TaskState.EXECUTING, 3: TaskState.FINISHED}


class _Entry:
    __slots__ = ("hid", "obj", "desc", "parent")

    def __init__(self, hid, obj, desc, parent=None):
        self.hid = hid
        self.obj = obj
        self.desc = desc
        self.parent = parent  # array-view element: the array it belongs to (kept alive)


def _element_of(buf, index):
    """The device operand of element ``index`` of an array view (access.py)."""
    if isinstance(buf, np.ndarray):
        if not -buf.shape[0] <= index < buf.shape[0]:
            raise IndexError(f"array view index {index} out of range")
        return buf[index:index + 1] if buf.ndim == 1 else buf[index]
    if isinstance(buf, (list, tuple)):
        return buf[index]
    raise ConfigurationError(
        f"array views need a numpy array or a list of device-movable objects, got {type(buf).__name__}")


class TaskViewer:
    """Reference to one inserted task (reference task.py:210-262)."""

    __slots__ = ("_graph", "_tid")

    def __init__(self, graph, tid):
        self._graph = graph
        self._tid = tid

    @property
    def task_id(self) -> int:
        return self._tid

    @property
    def state(self) -> TaskState:
        g = self._graph
        g._flush_batch()
        st = ctypes.c_int32(0)
        N.check(N.lib.sfx_task_state(g._h, self._tid, ctypes.byref(st)), g._h)
        return _STATE[st.value]

    def set_name(self, name: str) -> "TaskViewer":
        self._graph._names[self._tid] = name
        return self

    def wait(self, timeout=None) -> None:
        g = self._graph
        g._flush_batch()
        rc = N.lib.sfx_wait_task(g._h, self._tid, -1.0 if timeout is None else float(timeout))
        if rc == N.TIMEOUT:
            raise TimeoutError(f"timed out waiting for {g._label(self._tid)}")
        if rc == N.ERR_ENGINE_FAILED:
            raise g._failure()
        N.check(rc, g._h)

    def get_value(self):
        """The value a Python device callable returned; built-in and native ops
        produce no host value (the reference raises ValueError then, task.py:241-262)."""
        self.wait()
        g = self._graph
        if self._tid in g._py_vals:
            return g._py_vals[self._tid]
        op = g._py_ops.get(self._tid)
        if op is not None:
            try:
                v = g._py_vals[self._tid] = ops_mod.result_of(op)
                return v
            except KeyError:
                pass
        raise ValueError(f"{self._graph._label(self._tid)} produced no value")


class TraceView:
    """Events of one graph as reference tuples (kind, t_ns, worker, tid, extra)."""

    def __init__(self, graph):
        self._graph = graph
        self.enabled = True

    def export_events(self) -> list:
        g = self._graph
        g._flush_batch()
        n = ctypes.c_uint64(0)
        N.check(N.lib.sfx_trace(g._h, g._gid, None, 0, ctypes.byref(n)), g._h)
        buf = (N.Event * max(n.value, 1))()
        N.check(N.lib.sfx_trace(g._h, g._gid, buf, n.value, ctypes.byref(n)), g._h)
        t0 = g._t0
        out = []
        for e in buf[: n.value]:
            extra = e.extra if e.kind in (N.EV_STAGE_BEGIN, N.EV_STAGE_END) else None
            out.append((N.EV_NAMES[e.kind], e.t_ns - t0, e.worker, e.tid, extra))
        out.sort(key=lambda ev: ev[1])
        return out


class TaskGraph:
    """Sequential task flow over declared data accesses, executed on B200s."""

    def __init__(self, speculation: bool = False, trace: bool = True, history: bool = True):
        """``history=False`` (an extension): finished tasks and passed slots are
        retired by the runtime, so a long-running graph has bounded memory; the
        dot export / edges then only cover what is still live."""
        if speculation:
            raise SpeculationError(
                "speculative execution is not part of the GPU path (the reference also rejects "
                "device callables in speculative tasks, speculation.py:140-143)")
        self.engine = None
        self._h = None
        self._gid = None
        self._entries = {}  # id(obj) (or (id(obj), element)) -> _Entry
        self._hid_by_id = {}  # id(obj) -> hid of whole objects (the native fast path's lookup)
        self._hval = None
        self._by_hid = {}
        self._names = {}
        self._py_ops = {}   # tid -> Op of a Python device callable (get_value)
        self._py_vals = {}  # tid -> its value, once fetched
        self._name_ranges = []  # (first tid, count, name) of array submissions
        self._tids = []
        self._tid_ranges = []   # (first tid, count) of array submissions
        self._inserter_ident = None
        self._batch = None
        self._desc_buf = ctypes.create_string_buffer(96)
        self._acc_cap = 8
        self._acc_buf = ctypes.create_string_buffer(16 * self._acc_cap)
        self._t0 = time.perf_counter_ns()
        self.trace = TraceView(self)
        self.trace.enabled = trace
        self.speculation_enabled = False
        self.comm = None
        self.history = history

    def set_trace(self, enabled: bool) -> "TaskGraph":
        """Switch event recording on or off for the tasks inserted from now on."""
        self.trace.enabled = bool(enabled)
        if self.engine is not None:
            N.check(N.lib.sfx_graph_option(self._h, self._gid, b"trace", 1 if enabled else 0), self._h)
        return self

    # -- inter-process communication (graph.py:264-284, comms.py) -------------
    def use_comm(self, comm) -> "TaskGraph":
        """Bind to a communicator (comms.TorchComm) for send/recv/broadcast tasks."""
        if self.comm is not None and self.comm is not comm:
            raise ConfigurationError("graph is already bound to a communicator")
        self.comm = comm
        comm.graphs.append(self)
        return self

    def send(self, obj, dest: int, tag: int) -> "TaskViewer":
        from .comms import comm_send

        return comm_send(self, obj, dest, tag)

    def recv(self, obj, src: int, tag: int) -> "TaskViewer":
        from .comms import comm_recv

        return comm_recv(self, obj, src, tag)

    def broadcast(self, obj, root: int) -> "TaskViewer":
        from .comms import comm_broadcast

        return comm_broadcast(self, obj, root)

    # -- attachment (graph.py:57-64) -----------------------------------------
    def compute_on(self, engine) -> "TaskGraph":
        if self.engine is not None:
            raise ConfigurationError("graph is already attached to an engine")
        gid = ctypes.c_uint32(0)
        N.check(N.lib.sfx_graph_create(engine._h, ctypes.byref(gid)), engine._h)
        self.engine = engine
        self._h = engine._h
        self._hval = engine._h.value  # raw runtime pointer for the fast submit path
        self._gid = gid.value
        if not self.history:
            N.check(N.lib.sfx_graph_option(engine._h, self._gid, b"history", 0), engine._h)
        if not self.trace.enabled:  # TaskGraph(trace=False): no event recording (reference graph.py:34)
            N.check(N.lib.sfx_graph_option(engine._h, self._gid, b"trace", 0), engine._h)
        engine.adopt(self)
        self._t0 = time.perf_counter_ns()
        return self

    # -- registration (graph.py:68-73, handles.py:140-182) --------------------
    def _register(self, obj, key=None, parent=None) -> _Entry:
        desc = memory.describe(obj)
        hid = _next_hid()
        N.check(N.lib.sfx_register(self._h, self._gid, hid, desc.ptr, desc.nbytes, desc.rows, desc.cols,
                                   desc.ld, desc.dtype), self._h)
        e = _Entry(hid, obj, desc, parent)
        self._entries[id(obj) if key is None else key] = e
        if key is None:
            self._hid_by_id[id(obj)] = hid
        self._by_hid[hid] = e
        return e

    def element_hid(self, buf, index) -> int:
        """Handle of element ``index`` of ``buf`` (an array-view access), registered
        on first use under the identity (buf, index) -- reference graph.py:140-148."""
        key = (id(buf), int(index))
        e = self._entries.get(key)
        if e is None:
            if self.engine is None:
                raise ConfigurationError("attach the graph to an engine before inserting")
            e = self._register(_element_of(buf, int(index)), key=key, parent=buf)
        return e.hid

    def register(self, obj, nbytes: int = 0):
        if self.engine is None:
            raise ConfigurationError("attach the graph to an engine before registering")
        if id(obj) in self._entries:
            raise RegistrationError(f"object {type(obj).__name__} is already registered")
        return self._register(obj).hid

    def unregister(self, obj) -> None:
        e = self._entries.get(id(obj))
        if e is None:
            raise RegistrationError("object is not registered")
        self._flush_batch()
        N.check(N.lib.sfx_unregister(self._h, e.hid), self._h)
        del self._entries[id(obj)]
        self._hid_by_id.pop(id(obj), None)
        del self._by_hid[e.hid]

    def hid_of(self, obj) -> int:
        e = self._entries.get(id(obj))
        if e is None:
            if self.engine is None:
                raise ConfigurationError("attach the graph to an engine before inserting")
            e = self._register(obj)
        return e.hid

    def place(self, obj, device: int) -> None:
        """Owner hint for the locality-aware scheduler (e.g. 2-D block-cyclic)."""
        N.check(N.lib.sfx_set_home(self._h, self.hid_of(obj), int(device)), self._h)

    # -- insertion (graph.py:77-166) -------------------------------------------
    def task(self, *accesses, host=None, device=None, priority: int = 0, name=None):
        # native fast path (csrc/pyext/sfxfast.c): every object already registered,
        # no array views -> access codes, handle ids, a task id and the submit in C;
        # anything else (first use, views, errors) takes the Python path below
        pyop = None
        if device is not None and device.__class__ is not ops_mod.Op and callable(device):
            # a Python device callable, as in the reference (engine.py:144-149): a user op
            device = pyop = ops_mod.python_callable(device)
        if _fast_task is not None and host is None and self._hval is not None and self._batch is None:
            tid = _fast_task(self._hval, self._gid, self._hid_by_id, self._tids, accesses, device, priority)
            if tid > 0:
                if name is not None:
                    self._names[tid] = name
                if pyop is not None:
                    self._py_ops[tid] = pyop
                return TaskViewer(self, tid)
            if tid < -1:
                N.check(tid, self._h)
        if __debug__:
            ident = threading.get_ident()
            if self._inserter_ident != ident:
                assert self._inserter_ident is None, "tasks must be inserted by a single thread"
                self._inserter_ident = ident
        if self.engine is None:
            raise ConfigurationError("attach the graph to an engine before inserting")
        if device.__class__ is not ops_mod.Op:
            if device is None:
                if host is not None:
                    raise ConfigurationError(
                        "host callables run on the CPU oracle only: the GPU engine has no CPU fallback; "
                        "pass device=<paper_2308_15964_b200.ops op>")
                raise ConfigurationError("a task needs a host or device callable")
            if not isinstance(device, ops_mod.Op):
                raise ConfigurationError(
                    f"device= must be a registered op (paper_2308_15964_b200.ops), got {device!r}")
        hids = []
        modes = []
        entries = self._entries
        for spec in accesses:
            if spec.__class__ is not AccessSpec:
                if not isinstance(spec, AccessSpec):
                    raise ConfigurationError(f"accesses must be built with the access helpers, got {spec!r}")
            code = _MODE_CODE[spec.mode]
            if spec.view is not None:  # one handle per selected element (graph.py:140-148)
                for element in spec.view:
                    hid = self.element_hid(spec.obj, element)
                    if hid in hids:
                        raise DuplicateAccessError(f"task declares element {element} twice")
                    hids.append(hid)
                    modes.append(code)
                continue
            e = entries.get(id(spec.obj))
            hid = e.hid if e is not None else self.hid_of(spec.obj)
            if hid in hids:
                raise DuplicateAccessError(f"task declares {type(spec.obj).__name__} twice")
            hids.append(hid)
            modes.append(code)
        tid = _next_tid()
        if name is not None:
            self._names[tid] = name
        self._tids.append(tid)
        if pyop is not None:
            self._py_ops[tid] = pyop
        self._submit_one(tid, device, priority, hids, modes)
        return TaskViewer(self, tid)

    def _submit_one(self, tid, op, priority, hids, modes, dev_hint=-1):
        if self._batch is not None:
            self._batch.append((tid, op, priority, hids, modes, dev_hint))
            return
        if _fast_submit1 is not None:
            rc = _fast_submit1(self._hval, self._gid, tid, op.code, int(priority), dev_hint, op.fparam, op.iparam,
                               hids, modes)
            if rc < 0:
                N.check(rc, self._h)
            return
        # one struct.pack_into per descriptor into reused buffers (ctypes field
        # assignment costs ~10x more per task)
        n = len(hids)
        if n > self._acc_cap:
            self._acc_cap = max(n, 2 * self._acc_cap)
            self._acc_buf = ctypes.create_string_buffer(16 * self._acc_cap)
        fp, ip = op.fparam, op.iparam
        _DESC.pack_into(self._desc_buf, 0, tid, self._gid, op.code, int(priority), dev_hint, n, 0,
                        fp[0], fp[1], fp[2], fp[3], ip[0], ip[1], ip[2], ip[3])
        buf = self._acc_buf
        for k in range(n):
            _ACC.pack_into(buf, 16 * k, hids[k], modes[k], 0)
        rc = N.lib.sfx_submit(self._h, 1, self._desc_buf, buf)
        if rc < 0:
            N.check(rc, self._h)

    def submit_arrays(self, ops_codes, fparams, iparams, priorities, n_access, acc_hids, acc_modes,
                      devices=None, names=None) -> np.ndarray:
        """Vectorised insertion of many tasks in one call (same semantics as a loop of ``task``).

        Arrays are per task (op code, 4 fparams, 4 iparams, priority, access
        count) plus the flattened access list.  Returns the task ids.
        """
        self._flush_batch()
        n = len(ops_codes)
        descs = np.zeros(n, dtype=TASK_DTYPE)
        first = _reserve_tids(n)
        tids = np.arange(first, first + n, dtype=np.uint64)
        descs["tid"] = tids
        descs["graph"] = self._gid
        descs["op"] = ops_codes
        descs["priority"] = priorities
        descs["device"] = -1 if devices is None else devices
        descs["n_access"] = n_access
        descs["fparam"] = fparams
        descs["iparam"] = iparams
        acc = np.zeros(len(acc_hids), dtype=ACCESS_DTYPE)
        acc["hid"] = acc_hids
        acc["mode"] = acc_modes
        N.check(N.lib.sfx_submit(self._h, n, descs.ctypes.data, acc.ctypes.data if len(acc) else None), self._h)
        self._tid_ranges.append((first, n))
        if isinstance(names, str):  # one name for the whole block
            self._name_ranges.append((first, n, names))
        elif names is not None:
            for t, nm in zip(tids.tolist(), names):
                if nm is not None:
                    self._names[t] = nm
        return tids

    @contextlib.contextmanager
    def batch(self):
        """Buffer insertions and submit them in one native call on exit."""
        outer = self._batch is not None
        if not outer:
            self._batch = []
        try:
            yield self
        finally:
            if not outer:
                self._flush_batch()

    @contextlib.contextmanager
    def gated(self):
        """Insert with the executors held, like the reference's gate task
        (tests/conftest.py:184-203): the slot layout is then exactly the static one."""
        self.engine.pause()
        try:
            with self.batch():
                yield self
        finally:
            self.engine.resume()

    def _flush_batch(self):
        if not self._batch:
            if self._batch is not None:
                self._batch = None
            return
        batch = self._batch
        self._batch = None
        n = len(batch)
        total = sum(len(b[3]) for b in batch)
        descs = bytearray(_DESC.size * n)
        acc = bytearray(_ACC.size * max(total, 1))
        gid = self._gid
        pack_d, pack_a = _DESC.pack_into, _ACC.pack_into
        dsz, asz = _DESC.size, _ACC.size
        k = 0
        for i, (tid, op, prio, hids, modes, dev) in enumerate(batch):
            fp, ip = op.fparam, op.iparam
            pack_d(descs, i * dsz, tid, gid, op.code, int(prio), dev, len(hids), 0,
                   fp[0], fp[1], fp[2], fp[3], ip[0], ip[1], ip[2], ip[3])
            for h, m in zip(hids, modes):
                pack_a(acc, k * asz, h, m, 0)
                k += 1
        dbuf = (ctypes.c_char * len(descs)).from_buffer(descs)
        abuf = (ctypes.c_char * len(acc)).from_buffer(acc)
        N.check(N.lib.sfx_submit(self._h, n, dbuf, abuf), self._h)

    # -- waiting (graph.py:199-217) --------------------------------------------
    def _failure(self) -> EngineFailedError:
        code = ctypes.c_int(0)
        msg = ctypes.create_string_buffer(1024)
        N.lib.sfx_failure(self._h, ctypes.byref(code), msg, 1024)
        text = msg.value.decode(errors="replace")
        cause = N.error_for(code.value, text)
        if code.value == N.ERR_USER:
            user = ops_mod.take_error()  # the callable's own exception
            if user is not None:
                cause = user
                text = f"{text}: {type(user).__name__}: {user}"
        agent = getattr(self.engine, "_comm_agent", None)
        if agent is not None and agent.error is not None:
            cause = agent.error  # a communication task failed (e.g. CommProtocolError)
        err = EngineFailedError(f"a task failed: {text}")
        err.__cause__ = cause
        return err

    def wait_all(self, timeout=None) -> bool:
        if self.engine is None:
            return True
        self._flush_batch()
        rc = N.lib.sfx_wait_all(self._h, self._gid, -1.0 if timeout is None else float(timeout))
        if rc == N.TIMEOUT:
            return False
        if rc == N.ERR_ENGINE_FAILED:
            raise self._failure()
        N.check(rc, self._h)
        return True

    # -- device flush (graph.py:258-260) -----------------------------------------
    def flush_to_host(self, obj, keep_device: bool = False, element=None) -> TaskViewer:
        """Insert a flush of ``obj`` (or of its array-view ``element``) to its host buffer.

        Default = the reference's semantics: a host write, so every device copy
        is dropped afterwards.  ``keep_device=True`` only cleans the dirty copy
        (read-mode flush) and keeps device copies valid.
        """
        self._flush_batch()
        hid = self.hid_of(obj) if element is None else self.element_hid(obj, element)
        tid = _next_tid()
        self._names[tid] = "flush"
        self._tids.append(tid)
        N.check(N.lib.sfx_flush(self._h, self._gid, tid, hid, 0 if keep_device else 1), self._h)
        return TaskViewer(self, tid)

    def flush_all(self, keep_device: bool = True) -> None:
        for key, e in list(self._entries.items()):
            if isinstance(key, tuple):
                self.flush_to_host(e.parent, keep_device=keep_device, element=key[1])
            else:
                self.flush_to_host(e.obj, keep_device=keep_device)

    # -- export -----------------------------------------------------------------
    def _label(self, tid) -> str:
        nm = self._names.get(tid)
        if nm is None:
            for first, n, rn in self._name_ranges:
                if first <= tid < first + n:
                    return rn
        return nm or f"task{tid}"

    def all_task_ids(self) -> list:
        ids = list(self._tids)
        for first, n in self._tid_ranges:
            ids.extend(range(first, first + n))
        return sorted(ids)

    def edges(self) -> list:
        """Successor edges (src tid, dst tid, hid), one per handle pair (trace.py:94-102)."""
        self._flush_batch()
        n = ctypes.c_uint64(0)
        N.check(N.lib.sfx_edges(self._h, self._gid, None, None, None, 0, ctypes.byref(n)), self._h)
        m = max(n.value, 1)
        src = np.zeros(m, np.uint64)
        dst = np.zeros(m, np.uint64)
        hid = np.zeros(m, np.uint64)
        N.check(N.lib.sfx_edges(self._h, self._gid, src.ctypes.data, dst.ctypes.data, hid.ctypes.data, m,
                                ctypes.byref(n)), self._h)
        k = n.value
        return list(zip(src[:k].tolist(), dst[:k].tolist(), hid[:k].tolist()))

    def generate_dot(self, path=None, show_deps: bool = False) -> str:
        from .trace import generate_dot

        return generate_dot(self, path, show_deps)

    def generate_trace_svg(self, path=None, show_dep_arrows: bool = False, out=None) -> str:
        from .trace import generate_trace_svg

        return generate_trace_svg(self, path, show_dep_arrows, out)
