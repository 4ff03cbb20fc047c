"""Compute engines over B200 devices (drop-in for reference src/engine.py:38-285).

``create_engine(WorkerTeam.of_host_and_device_workers(devices=N,
workers_per_device=K))`` creates one native runtime driving N GPUs with K
CUDA streams each (a reference "device worker" maps onto a stream).  Host
workers are accepted for signature compatibility but the GPU engine never
runs a task on the CPU: host callables belong to the oracle.

Differences from the reference, by design:

* ``device_memory`` defaults to "most of the GPU" (free HBM minus a reserve)
  instead of 16 MiB -- a single 1024x1024 FP64 tile is 8 MiB.
* ``backend="sim"`` selects host-memory simulated devices for bookkeeping
  tests on machines without a GPU; it refuses every tile op.
* ``window`` bounds in-flight tasks per device (run-ahead of the launcher).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native as N
from .errors import ConfigurationError
from .scheduler import DEVICE, HOST, WorkerKind, native_policy


class WorkerTeam:
    """A team description: list of (WorkerKind, count) pairs (engine.py:38-68)."""

    def __init__(self, spec):
        self.spec = [(kind, int(count)) for kind, count in spec]
        if sum(count for _, count in self.spec) <= 0:
            raise ConfigurationError("a worker team needs at least one worker")

    def kinds(self):
        for kind, count in self.spec:
            for _ in range(count):
                yield kind

    def device_indexes(self):
        return sorted({kind.device for kind, _ in self.spec if kind.kind == DEVICE})

    def workers_per_device(self) -> int:
        counts = [count for kind, count in self.spec if kind.kind == DEVICE]
        return max(counts) if counts else 0

    @staticmethod
    def of_host_workers(n: int) -> "WorkerTeam":
        return WorkerTeam([(WorkerKind.host(), n)])

    @staticmethod
    def of_host_and_device_workers(devices: int = 1, host_workers=None,
                                   workers_per_device: int = 1) -> "WorkerTeam":
        if host_workers is None:
            host_workers = max(1, (os.cpu_count() or 2) - devices)
        spec = [(WorkerKind.host(), host_workers)]
        for i in range(devices):
            spec.append((WorkerKind.device_worker(i), workers_per_device))
        return WorkerTeam(spec)

    @staticmethod
    def of_devices(devices: int = 1, streams_per_device: int = 8) -> "WorkerTeam":
        """GPU-only team: ``devices`` GPUs with ``streams_per_device`` streams each."""
        return WorkerTeam([(WorkerKind.device_worker(i), streams_per_device) for i in range(devices)])


class ComputeEngine:
    """A native runtime over the team's devices, serving any number of graphs."""

    def __init__(self, team, scheduler=None, device_memory=None, *, backend: str = "cuda",
                 trace: bool = True, window: int = 0, ordinals=None, arena_align: int = 0,
                 group_max: int = 32, kernel_timing: bool = False, deterministic: bool = False):
        if isinstance(team, (list, tuple)):
            team = WorkerTeam(team)
        devices = team.device_indexes()
        if not devices:
            raise ConfigurationError(
                "the GPU engine needs device workers (WorkerTeam.of_host_and_device_workers); "
                "host-only teams run on the CPU oracle")
        if backend not in ("cuda", "sim"):
            raise ConfigurationError(f"unknown backend {backend!r}")
        self.team = team
        self.backend = backend
        self.ndev = len(devices)
        self.streams_per_device = max(1, team.workers_per_device())
        self.policy = native_policy(scheduler)
        self.trace_enabled = trace
        flags = N.FLAG_TRACE if trace else 0
        if kernel_timing:
            flags |= N.FLAG_KTIME  # stats(): timed_groups / timed_tasks / timed_ns
        if backend == "sim":
            flags |= N.FLAG_SIM
        if arena_align:
            lg = int(arena_align).bit_length() - 1
            if 1 << lg != arena_align:
                raise ConfigurationError("arena_align must be a power of two")
            flags |= lg << 8
        if backend == "cuda":
            have = N.device_count()
            if have == 0:
                raise ConfigurationError(
                    "no CUDA device is visible: the GPU engine has no CPU fallback "
                    "(use backend='sim' for bookkeeping tests, or the oracle for CPU runs)")
        if ordinals is None:
            ordinals = list(range(self.ndev))
        ords = (ctypes.c_int * self.ndev)(*ordinals)
        arenas = None
        if device_memory is not None:
            sizes = device_memory if isinstance(device_memory, (list, tuple)) else [device_memory] * self.ndev
            arenas = (ctypes.c_uint64 * self.ndev)(*[int(s) for s in sizes])
        self.device_memory = device_memory
        handle = ctypes.c_void_p()
        N.check(N.lib.sfx_create(self.ndev, ords, self.streams_per_device, arenas, self.policy,
                                 flags, int(window), ctypes.byref(handle)))
        self._h = handle
        self.set_option("group_max", group_max)
        if deterministic:  # no order-dependent FP64 accumulation (runtime option, sfx.h)
            self.set_option("deterministic", 1)
        # runtime knobs from the environment (experiments): SFX_OPT_<KEY>=<int>
        for key, value in os.environ.items():
            if key.startswith("SFX_OPT_"):
                self.set_option(key[8:].lower(), int(value))
        self.graphs = []
        self._stopped = False

    # -- graph attachment (engine.py:202-204) --------------------------------
    def adopt(self, graph) -> None:
        self.graphs.append(graph)

    def kind_classes(self) -> set:
        return {DEVICE}

    # -- control --------------------------------------------------------------
    def set_option(self, key: str, value: int) -> None:
        """Runtime knobs: ``group_max`` (grouped launches), ``window`` (in-flight tasks)."""
        N.check(N.lib.sfx_set_option(self._h, key.encode(), int(value)), self._h)

    def pause(self) -> None:
        """Hold the executors (the gate task of the reference's gated insertion)."""
        N.check(N.lib.sfx_pause(self._h), self._h)

    def resume(self) -> None:
        N.check(N.lib.sfx_resume(self._h), self._h)

    def stop(self) -> None:
        if not self._stopped:
            self._stopped = True
            agent = getattr(self, "_comm_agent", None)
            if agent is not None:
                agent.stop()
            N.lib.sfx_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc_info):
        self.stop()
        return False

    def __del__(self):
        try:
            self.stop()
        except Exception:
            pass

    # -- introspection --------------------------------------------------------
    def worker_count(self, kind_class=None) -> int:
        n = self.ndev * self.streams_per_device
        if kind_class in (None, DEVICE):
            return n
        return 0

    def worker_stride(self) -> int:
        """Trace worker ids are device * stride + stream (all stream classes of a GPU:
        normal, high-priority, cooperative, prefetch)."""
        n = self.streams_per_device
        urgent = max(2, n // 4) if n >= 2 else 0
        coop = 0 if self.backend == "sim" else 2
        return n + urgent + coop

    def stats(self, dev: int = 0) -> dict:
        st = N.DevStats()
        N.check(N.lib.sfx_stats(self._h, dev, ctypes.byref(st)), self._h)
        return st.as_dict()

    def resident(self, dev: int = 0) -> set:
        n = ctypes.c_uint64(0)
        N.check(N.lib.sfx_resident(self._h, dev, None, 0, ctypes.byref(n)), self._h)
        buf = np.zeros(max(n.value, 1), dtype=np.uint64)
        N.check(N.lib.sfx_resident(self._h, dev, buf.ctypes.data, n.value, ctypes.byref(n)), self._h)
        return set(int(x) for x in buf[: n.value])

    def block_state(self, hid: int, dev: int = 0):
        st = ctypes.c_int32(0)
        hv = ctypes.c_int32(0)
        N.check(N.lib.sfx_block_state(self._h, hid, dev, ctypes.byref(st), ctypes.byref(hv)), self._h)
        return {"present": bool(st.value & 4), "valid": bool(st.value & 1), "dirty": bool(st.value & 2),
                "host_valid": bool(hv.value)}

    def live(self) -> dict:
        """Runtime-wide live Task objects and slots, and tasks retired so far."""
        t, sl, r = ctypes.c_uint64(0), ctypes.c_uint64(0), ctypes.c_uint64(0)
        N.check(N.lib.sfx_live(self._h, ctypes.byref(t), ctypes.byref(sl), ctypes.byref(r)), self._h)
        return {"tasks": t.value, "slots": sl.value, "retired": r.value}

    def violations(self) -> int:
        n = ctypes.c_uint64(0)
        N.check(N.lib.sfx_violations(self._h, ctypes.byref(n)), self._h)
        return n.value


def create_engine(team, scheduler=None, device_memory=None, **kw) -> ComputeEngine:
    return ComputeEngine(team, scheduler, device_memory, **kw)


def attach_graph(graph, engine: ComputeEngine) -> None:
    graph.compute_on(engine)


def fp64_peak(ordinal: int = 0):
    """Measured FP64 DMMA peak (TFLOP/s) and the device's max SM clock (MHz)."""
    t = ctypes.c_double(0)
    mhz = ctypes.c_double(0)
    N.check(N.lib.sfx_fp64_peak(ordinal, ctypes.byref(t), ctypes.byref(mhz)))
    return t.value, mhz.value


def fp64_dfma_peak(ordinal: int = 0) -> float:
    """Measured FP64 pipe (DFMA) peak in TFLOP/s (2 flop per FMA)."""
    t = ctypes.c_double(0)
    N.check(N.lib.sfx_fp64_dfma_peak(ordinal, ctypes.byref(t)))
    return t.value


HOST_KIND = HOST
