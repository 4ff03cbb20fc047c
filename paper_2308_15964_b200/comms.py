"""Multi-process communication tasks: send / recv / broadcast between graph
instances of different processes.

Reference: ``src/comms.py`` -- ``CommInstance`` / ``CommAgent`` (303-483) over an
in-process ``InProcessUniverse`` (206-276), the insertion entry points
``comm_send`` / ``comm_recv`` / ``comm_broadcast`` (541-599), the two-part wire
message (a 16-byte ``<iiQ`` header -- tag, source, payload size -- then the
payload, 39 and 415-427), FIFO matching per (source, tag) and the hidden
broadcast tag ``1 << 30`` (40, 582).

Here the ranks are PROCESSES (one per GPU or per node) and the transport is
``torch.distributed`` point-to-point (gloo over TCP; any backend whose
isend/irecv accept CPU tensors).  A communication task is a native
``SFX_OP_EXTERN`` task: the runtime orders it with the other tasks by its
declared access (send = read, recv = write), makes the object's host buffer
current when it becomes ready (a dirty GPU copy is fetched home first; a
receive drops the GPU copies), and hands it to this module's agent thread
through ``sfx_extern_poll``; the agent moves the bytes straight from / into
the object's host buffer and finishes the task with ``sfx_extern_done``,
which releases its successors (a GPU task reading a received tile stages it
from the host buffer).  Message matching follows the reference: per
(peer, tag) channel, receives match sends in posting order.
"""

from __future__ import annotations

import ctypes
import logging
import threading
from collections import deque

import numpy as np

from . import _native as N
from .access import AccessMode
from .errors import CommProtocolError, ConfigurationError, SerializationError

log = logging.getLogger("paper_2308_15964_b200")

BCAST_FLAG = 1 << 30  # reference comms.py:40
MAX_TAG = BCAST_FLAG  # reference comms.py:41


def payload_view(obj) -> np.ndarray:
    """The object's host buffer as a flat writable uint8 array (the payload).

    Tiers of the reference's ``resolve_tier`` (comms.py:135-155) that exist on
    this path: numpy arrays (tiles, particle blocks), ``Cell`` (8-byte buffer),
    writable buffers (bytearray).  Anything else raises SerializationError.
    """
    buf = getattr(obj, "__sfx_buffer__", None)
    if buf is not None:
        obj = buf()
    if isinstance(obj, np.ndarray):
        if not obj.flags.c_contiguous:
            raise SerializationError("communication needs a contiguous array")
        return obj.reshape(-1).view(np.uint8)
    try:
        mv = memoryview(obj)
    except TypeError:
        raise SerializationError(f"cannot transfer a {type(obj).__name__}") from None
    if mv.readonly or not mv.contiguous:
        raise SerializationError(f"cannot transfer a read-only or non-contiguous {type(obj).__name__}")
    return np.frombuffer(mv.cast("B"), dtype=np.uint8)


class TorchComm:
    """One rank of a torch.distributed process group used as the communicator
    (replaces ``InProcessUniverse.instances[rank]``, reference comms.py:206-276).

    ``torch.distributed.init_process_group`` must have been called (e.g. by
    torchrun, backend "gloo").  ``max_message_size`` mirrors the reference's
    universe limit: larger payloads poison the engine with CommProtocolError.
    """

    def __init__(self, group=None, max_message_size: int = 1 << 40):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise ConfigurationError("TorchComm needs torch.distributed.init_process_group first")
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.max_message_size = int(max_message_size)
        self._bcast_seq = 0
        self.graphs = []

    def next_bcast_seq(self) -> int:
        seq = self._bcast_seq
        self._bcast_seq += 1
        return seq


class _Op:
    __slots__ = ("kind", "obj", "peer", "tag", "comm", "tid", "dests")

    def __init__(self, kind, obj, peer, tag, comm):
        self.kind, self.obj, self.peer, self.tag, self.comm = kind, obj, peer, tag, comm
        self.tid = 0
        self.dests = ()


class CommAgent:
    """One agent per engine (reference CommAgent, comms.py:303-483): takes ready
    communication tasks from the runtime and finishes them in the runtime once
    their transfer is done.

    Each (kind, peer, tag) channel is served by its own thread, in posting order
    (receives match sends FIFO per channel, reference comms.py:404-411,455-460);
    a channel thread blocks in the transport (gloo completes point-to-point work
    only through ``wait()``) and exits when its queue is empty.
    """

    def __init__(self, engine):
        self.engine = engine
        self._ops = {}  # tid -> _Op (registered before the task is submitted)
        self._lock = threading.Lock()
        self._stop = False
        self._channels = {}  # (kind, peer, tag) -> deque of ops; present while a thread serves it
        self.error = None
        self.wakeups = 0
        self._thread = threading.Thread(target=self._loop, name="sfx-comm-agent", daemon=True)
        self._thread.start()

    def register(self, tid: int, op: _Op) -> None:
        op.tid = tid
        with self._lock:
            self._ops[tid] = op

    def stop(self) -> None:
        self._stop = True
        self._thread.join(timeout=5)
        with self._lock:
            pending = [op for q in self._channels.values() for op in q if op.kind in ("recv", "bcast_recv")]
        if pending:
            log.warning("communication agent stopped with %d pending receive(s)", len(pending))

    # -- transfers (two-part message, reference comms.py:415-427) --------------
    @staticmethod
    def _stage(op: _Op):
        """A private copy of a send's payload (the task's buffer is free after it)."""
        import torch

        payload = torch.from_numpy(payload_view(op.obj)).clone()
        if payload.numel() > op.comm.max_message_size:
            raise CommProtocolError(f"message of {payload.numel()} bytes exceeds the limit "
                                    f"{op.comm.max_message_size}")
        return payload

    @staticmethod
    def _transfer(op: _Op, staged=None) -> None:
        import torch

        dist, comm = op.comm.dist, op.comm
        payload = staged if staged is not None else torch.from_numpy(payload_view(op.obj))
        nbytes = payload.numel()
        if op.kind in ("send", "bcast_root"):
            if nbytes > comm.max_message_size:
                raise CommProtocolError(f"message of {nbytes} bytes exceeds the limit {comm.max_message_size}")
            header = torch.tensor([op.tag, comm.rank, nbytes], dtype=torch.int64)
            works = []
            for d in (op.dests if op.kind == "bcast_root" else (op.peer,)):
                works.append(dist.isend(header, d, group=comm.group, tag=op.tag))
                works.append(dist.isend(payload, d, group=comm.group, tag=op.tag))
            for w in works:
                w.wait()
            return
        header = torch.zeros(3, dtype=torch.int64)
        dist.irecv(header, op.peer, group=comm.group, tag=op.tag).wait()
        _tag, src, size = (int(x) for x in header.tolist())
        if size > comm.max_message_size:
            raise CommProtocolError(f"message of {size} bytes exceeds the limit {comm.max_message_size}")
        if size != nbytes or src != op.peer:
            # drain the payload so the channel stays aligned, then fail
            scratch = torch.empty(size, dtype=torch.uint8)
            dist.irecv(scratch, op.peer, group=comm.group, tag=op.tag).wait()
            raise CommProtocolError(f"message from rank {src} with {size} bytes does not fit the receive "
                                    f"buffer ({nbytes} bytes from rank {op.peer})")
        dist.irecv(payload, op.peer, group=comm.group, tag=op.tag).wait()

    def _serve(self, key) -> None:
        h = self.engine._h
        while True:
            with self._lock:
                q = self._channels[key]
                if not q or self._stop:
                    del self._channels[key]
                    return
                op = q[0]
            try:
                if op.kind in ("send", "bcast_root"):
                    # a send completes as soon as it is posted (reference comms.py:
                    # universe.put, then _complete): the payload is staged and the task
                    # finishes -- releasing its READ access -- before the transfer,
                    # which may wait for the peer's matching receive.  Otherwise a
                    # send(X) followed by recv(X) on both ranks would deadlock: each
                    # recv waits for its own send, each send for the peer's recv.
                    staged = self._stage(op)
                    if not self._stop:
                        N.lib.sfx_extern_done(h, op.tid, 0, None)
                    self._transfer(op, staged)
                else:
                    self._transfer(op)
                    if not self._stop:  # the runtime is gone once its engine stopped
                        N.lib.sfx_extern_done(h, op.tid, 0, None)
            except Exception as exc:  # noqa: BLE001 -- reported through the engine
                self.error = exc
                if not self._stop:
                    msg = f"{type(exc).__name__}: {exc}".encode()
                    if op.kind in ("send", "bcast_root"):
                        N.lib.sfx_fail(h, msg)  # the task already finished: poison directly
                    else:
                        N.lib.sfx_extern_done(h, op.tid, 1, msg)
            with self._lock:
                q.popleft()

    def _loop(self) -> None:
        h = self.engine._h
        buf = (ctypes.c_uint64 * 64)()
        n = ctypes.c_uint64(0)
        while not self._stop:
            N.lib.sfx_extern_poll(h, buf, 64, ctypes.byref(n), 0.05)
            if not n.value:
                continue
            self.wakeups += 1
            for k in range(n.value):
                with self._lock:
                    op = self._ops.pop(int(buf[k]))
                    key = (op.kind, op.peer, op.tag)
                    q = self._channels.get(key)
                    start = q is None
                    if start:
                        q = self._channels[key] = deque()
                    q.append(op)
                if start:
                    threading.Thread(target=self._serve, args=(key,), daemon=True,
                                     name=f"sfx-comm-{op.kind}-{op.peer}-{op.tag}").start()


def agent_for(engine) -> CommAgent:
    agent = getattr(engine, "_comm_agent", None)
    if agent is None:
        agent = CommAgent(engine)
        engine._comm_agent = agent
    return agent


# -- insertion entry points (reference comms.py:508-599) ----------------------

def _precheck(graph, obj, peer: int, tag: int):
    comm = graph.comm
    if comm is None:
        raise ConfigurationError("bind the graph to a communicator with use_comm before inserting "
                                 "communication tasks")
    if not 0 <= peer < comm.size:
        raise ConfigurationError(f"rank {peer} outside communicator of size {comm.size}")
    if not 0 <= tag < MAX_TAG:
        raise ConfigurationError(f"tag must be in [0, {MAX_TAG}), got {tag}")
    payload_view(obj)  # unresolvable objects fail at insertion (reference resolve_tier)
    return comm


def _insert(graph, op: _Op, mode: AccessMode, name: str):
    from .graph import TaskViewer, _MODE_CODE, _next_tid

    graph._flush_batch()
    hid = graph.hid_of(op.obj)
    tid = _next_tid()
    graph._names[tid] = name
    graph._tids.append(tid)
    agent_for(graph.engine).register(tid, op)
    graph._submit_one(tid, _EXTERN, 0, [hid], [_MODE_CODE[mode]])
    return TaskViewer(graph, tid)


class _ExternOp:
    code = N.OP_EXTERN
    fparam = (0.0, 0.0, 0.0, 0.0)
    iparam = (0, 0, 0, 0)
    name = "extern"


_EXTERN = _ExternOp()


def comm_send(graph, obj, dest: int, tag: int):
    comm = _precheck(graph, obj, dest, tag)
    return _insert(graph, _Op("send", obj, dest, tag, comm), AccessMode.READ, f"send->r{dest}#{tag}")


def comm_recv(graph, obj, src: int, tag: int):
    comm = _precheck(graph, obj, src, tag)
    return _insert(graph, _Op("recv", obj, src, tag, comm), AccessMode.WRITE, f"recv<-r{src}#{tag}")


def comm_broadcast(graph, obj, root: int):
    """Root fans out to every other rank under the hidden tag (reference 570-599)."""
    from . import ops

    comm = _precheck(graph, obj, root, 0)
    seq = comm.next_bcast_seq()
    if comm.size == 1:
        return graph.task(graph_read(obj), device=ops.noop, name=f"bcast#{seq}")
    if comm.rank == root:
        op = _Op("bcast_root", obj, root, BCAST_FLAG, comm)
        op.dests = tuple(r for r in range(comm.size) if r != root)
        return _insert(graph, op, AccessMode.READ, f"bcast#{seq}")
    return _insert(graph, _Op("bcast_recv", obj, root, BCAST_FLAG, comm), AccessMode.WRITE, f"bcast#{seq}")


def graph_read(obj):
    from .access import read

    return read(obj)
