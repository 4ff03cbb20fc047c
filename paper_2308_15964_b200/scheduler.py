"""Worker kinds and scheduling policies (reference src/scheduler.py:24-147).

In the reference, device workers are threads pulling from ONE shared DEVICE
queue (scheduler.py:71), so a task lands on whichever device worker pops it
first.  On the B200 path each device (GPU) has its own native ready queue
and a locality-aware placement decides the device when a task becomes ready
(owner of the written tile, else the device holding most operand bytes,
else the least loaded).  The policy inside each queue is the reference's:
FIFO (scheduler.py:66-94) or priority with FIFO ties (scheduler.py:97-126).

``FifoScheduler`` / ``PriorityScheduler`` / "fifo" / "prio" select the
native policy.  Custom Python ``Scheduler`` subclasses cannot run inside the
native executors; they are accepted only by the CPU oracle.
"""

from __future__ import annotations

import abc
from dataclasses import dataclass

from . import _native as N
from .errors import ConfigurationError

HOST = "host"
DEVICE = "device"


@dataclass(frozen=True)
class WorkerKind:
    """Classification of a worker: host, or device with an index."""

    kind: str
    device: int | None = None

    @staticmethod
    def host() -> "WorkerKind":
        return WorkerKind(HOST)

    @staticmethod
    def device_worker(index: int) -> "WorkerKind":
        return WorkerKind(DEVICE, index)

    def __str__(self):
        return self.kind if self.device is None else f"{self.kind}{self.device}"


class Scheduler(abc.ABC):
    """Marker base class mirroring the reference plugin contract."""

    native_policy = None


class FifoScheduler(Scheduler):
    native_policy = N.SCHED_FIFO


class PriorityScheduler(Scheduler):
    native_policy = N.SCHED_PRIO


_BY_NAME = {"fifo": N.SCHED_FIFO, "prio": N.SCHED_PRIO}


def native_policy(spec) -> int:
    """Accepts None, "fifo"/"prio", FifoScheduler/PriorityScheduler (class or instance)."""
    if spec is None:
        return N.SCHED_FIFO
    if isinstance(spec, str):
        try:
            return _BY_NAME[spec]
        except KeyError:
            raise ConfigurationError(
                f"unknown scheduler {spec!r}; expected one of {sorted(_BY_NAME)}") from None
    policy = getattr(spec, "native_policy", None)
    if policy is not None:
        return policy
    raise ConfigurationError(
        f"scheduler {spec!r} is a Python plugin; the GPU engine runs the native fifo/prio "
        "policies only (custom schedulers run on the CPU oracle)")
