#!/usr/bin/env python
"""Run one tiled workload through the public API for ncu captures.

    python tools/prof_workload.py gemm --n 4096 --b 512 --reps 3
    python tools/prof_workload.py cholesky --n 32768 --b 1024 --reps 1
    python tools/prof_workload.py particles --groups 8 --per 4096 --reps 1

Under ncu, select the kernel and the launch with -k / -s / -c, e.g.
    ncu --set full --clock-control none --import-source on -k regex:dgemm_dmma -s 20 -c 1 \
        -o gpurun_out/dgemm python tools/prof_workload.py gemm --n 8192 --b 512
Inputs are generated on the device (splitmix64), nothing is checked here:
parity lives in tests/.
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
    ap.add_argument("workload", choices=("gemm", "cholesky", "particles"))
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--b", type=int, default=512)
    ap.add_argument("--groups", type=int, default=16)
    ap.add_argument("--per", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--streams", type=int, default=16)
    ap.add_argument("--group-max", type=int, default=32)
    a = ap.parse_args()
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, a.streams), scheduler="prio", trace=False,
                           group_max=a.group_max, kernel_timing=True)
    g = sf.TaskGraph().compute_on(eng)
    if a.workload == "gemm":
        A, B, C = (alg.TiledMatrix(a.n, a.b) for _ in range(3))
        alg.insert_fill_uniform(g, A, 1)
        alg.insert_fill_uniform(g, B, 2)
        alg.insert_zero(g, C)
        g.wait_all()
        work, unit = alg.flops_gemm(a.n), "GFLOP/s"
        run = lambda: alg.insert_gemm(g, A, B, C)  # noqa: E731
    elif a.workload == "cholesky":
        M = alg.TiledMatrix(a.n, a.b, lower=True)
        work, unit = alg.flops_cholesky(a.n), "GFLOP/s"

        def run():
            alg.insert_fill_spd(g, M, 3)
            g.wait_all()
            alg.insert_cholesky(g, M)
    else:
        P = [sf.pinned_empty((4, a.per)) for _ in range(a.groups)]
        F = [sf.pinned_empty((4, a.per)) for _ in range(a.groups)]
        alg.insert_fill_particles(g, P, 4)
        for f in F:
            g.task(sf.write(f), device=sf.ops.zero())
        g.wait_all()
        work, unit = alg.interactions(a.groups * a.per), "interactions/s (x1e-9)"
        run = lambda: alg.insert_particles(g, P, F)  # noqa: E731
    for r in range(a.reps):
        t0 = time.perf_counter()
        run()
        g.wait_all()
        dt = time.perf_counter() - t0
        print(f"rep {r}: {dt * 1e3:.1f} ms  {work / dt / 1e9:.1f} {unit} (wall clock, includes insertion)")
    st = eng.stats(0)
    print({k: st[k] for k in ("kernel_launches", "groups", "timed_groups", "timed_tasks", "timed_ns", "busy_ns")})
    eng.stop()


if __name__ == "__main__":
    main()
