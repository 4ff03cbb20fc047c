#!/usr/bin/env python
"""Where a C2 step's time goes outside the DGEMM kernels (runtime trace, CUDA-event
timestamps on CLOCK_MONOTONIC, comparable with time.perf_counter_ns).

    python tools/step_gaps.py [--n 16384 --b 512 --streams 32 --group 32]

Prints: insertion time, delay from step start to the first kernel, from the
last kernel end to wait_all's return, and a per-2%-of-step histogram of how
many launch groups were running.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2308_15964_b200 as sf  # noqa: E402
from paper_2308_15964_b200 import algorithms as alg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--b", type=int, default=512)
    ap.add_argument("--streams", type=int, default=32)
    ap.add_argument("--group", type=int, default=32)
    ap.add_argument("--ktime", action="store_true", help="no trace: kernel-timing stats only (lower overhead)")
    a = ap.parse_args()
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, a.streams), scheduler="prio", trace=not a.ktime,
                           group_max=a.group, kernel_timing=a.ktime)
    A, B, C = (alg.TiledMatrix(a.n, a.b) for _ in range(3))
    g = sf.TaskGraph().compute_on(eng)
    alg.insert_fill_uniform(g, A, 1)
    alg.insert_fill_uniform(g, B, 2)
    alg.insert_zero(g, C)
    g.wait_all()
    for rep in range(3):
        eng.stats(0)
        t0 = time.perf_counter_ns()
        alg.insert_gemm(g, A, B, C)
        t_ins = time.perf_counter_ns()
        g.wait_all()
        t1 = time.perf_counter_ns()
        if a.ktime:
            st = eng.stats(0)
            print(f"step {(t1 - t0) / 1e6:.1f} ms  insertion {(t_ins - t0) / 1e6:.1f} ms  start->first kernel "
                  f"{(st['first_start_ns'] - t0) / 1e6:.2f} ms  last kernel->wait_all return "
                  f"{(t1 - st['last_end_ns']) / 1e6:.2f} ms  busy {st['busy_ns'] / 1e6:.1f} ms")
    if a.ktime:
        eng.stop()
        return
    ev = g.trace.export_events()
    base = g._t0
    spans = {}
    for kind, t, w, tid, _ in ev:
        if kind in ("TaskStart", "TaskEnd"):
            spans.setdefault(tid, [None, None, w])[0 if kind == "TaskStart" else 1] = t + base
    groups = {(s, e, w) for s, e, w in spans.values() if s and e}
    first = min(s for s, _, _ in groups)
    last = max(e for _, e, _ in groups)
    step = t1 - t0
    print(f"step {step / 1e6:.1f} ms  insertion {(t_ins - t0) / 1e6:.1f} ms  start->first kernel "
          f"{(first - t0) / 1e6:.2f} ms  last kernel->wait_all return {(t1 - last) / 1e6:.2f} ms  "
          f"groups {len(groups)}")
    nb = 50
    hist = [0.0] * nb
    for s, e, _ in groups:
        for k in range(nb):
            lo = t0 + step * k / nb
            hi = t0 + step * (k + 1) / nb
            ov = min(e, hi) - max(s, lo)
            if ov > 0:
                hist[k] += ov / (hi - lo)
    print("mean running groups per 2% of the step:", " ".join(f"{h:.1f}" for h in hist))
    eng.stop()


if __name__ == "__main__":
    main()
