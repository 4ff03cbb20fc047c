"""Spin-op durations and chain makespans on the GPU engine (overhead-protocol debugging)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2308_15964_b200 as sf  # noqa: E402

for trace in (False, True):
    for T in (1, 4, 16):
        eng = sf.create_engine(sf.WorkerTeam.of_devices(1, T), trace=trace, device_memory=1 << 26)
        N, D = 200, 1e-3
        g = sf.TaskGraph().compute_on(eng)
        cells = [sf.Cell(0) for _ in range(T)]
        for c in cells:
            g.task(sf.write(c), device=sf.ops.noop)
        g.wait_all()
        t0 = time.perf_counter()
        for i in range(N):
            for c in cells:
                g.task(sf.write(c), device=sf.ops.spin(int(D * 1e9)))
        g.wait_all()
        dt = time.perf_counter() - t0
        st = eng.stats(0)
        print(f"trace={trace} T={T}: {dt / N * 1e3:.3f} ms per chain step (D = {D * 1e3} ms), groups {st['groups']}",
              flush=True)
        eng.stop()
# one spin kernel alone, timed with torch events on a torch stream via a 1-stream engine
eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 1), trace=True, device_memory=1 << 26)
g = sf.TaskGraph().compute_on(eng)
c = sf.Cell(0)
for ns in (10_000, 100_000, 1_000_000):
    g.task(sf.write(c), device=sf.ops.spin(ns))
g.wait_all()
ev = g.trace.export_events()
st = {e[3]: e[1] for e in ev if e[0] == "TaskStart"}
en = {e[3]: e[1] for e in ev if e[0] == "TaskEnd"}
for tid in sorted(st):
    print("spin task", tid, "device time us", (en[tid] - st[tid]) / 1e3)
eng.stop()
