#!/usr/bin/env python
"""Sweep runtime knobs on the tiled Cholesky (device-resident, CUDA-event timed).

    python tools/chol_sweep.py --n 32768 --b 1024 [--reps 3]

Each line: knobs -> mean seconds and TFLOP/s of the factorization (fill excluded).
"""
from __future__ import annotations

import argparse
import itertools
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2308_15964_b200 as sf  # noqa: E402
from paper_2308_15964_b200 import algorithms as alg  # noqa: E402


def run(n, b, reps, streams, group, gps, prio, urgent, arena_gib=0.0):
    mem = int(arena_gib * 2 ** 30) if arena_gib else None
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, streams), scheduler="prio", trace=False, group_max=group,
                           device_memory=mem)
    eng.set_option("groups_per_stream", gps)
    if urgent is not None:
        eng.set_option("urgent_priority", urgent)
    M = alg.TiledMatrix(n, b, lower=True)
    g = sf.TaskGraph().compute_on(eng)
    ts = []
    for rep in range(reps + 1):
        alg.insert_fill_spd(g, M, 3)
        g.wait_all()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        alg.insert_cholesky(g, M, priorities={0: False, 1: True, 2: "critical", 3: "auto"}[prio])
        g.wait_all()
        e1.record()
        torch.cuda.synchronize()
        if rep:
            ts.append(e0.elapsed_time(e1) / 1e3)
    st = eng.stats(0)
    if arena_gib:
        print(f"  arena {arena_gib} GiB: evictions {st['evictions']}, write-backs {st['writebacks']}, "
              f"H2D {st['bytes_to_device'] / 2 ** 30:.1f} GiB, D2H {st['bytes_from_device'] / 2 ** 30:.1f} GiB "
              f"over {reps + 1} factorizations (+ fills)")
    eng.stop()
    t = statistics.mean(ts)
    return t, alg.flops_cholesky(n) / t / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--b", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--streams", default="16")
    ap.add_argument("--group", default="32")
    ap.add_argument("--gps", default="2")
    ap.add_argument("--prio", default="1", help="0 none, 1 column priorities, 2 critical-path only, 3 auto")
    ap.add_argument("--urgent", default="default")
    ap.add_argument("--arena-gib", type=float, default=0.0, help="cap the device arena (LRU tile cache) size")
    a = ap.parse_args()
    ints = lambda s: [int(x) for x in s.split(",")]  # noqa: E731
    urg = [None if u == "default" else int(u) for u in a.urgent.split(",")]
    for st, gr, gps, pr, ur in itertools.product(ints(a.streams), ints(a.group), ints(a.gps), ints(a.prio), urg):
        t, tf = run(a.n, a.b, a.reps, st, gr, gps, pr, ur, a.arena_gib)
        print(f"streams={st} group={gr} groups_per_stream={gps} prio={pr} urgent={ur} arena={a.arena_gib or 'all'} "
              f"tiles_per_cta="
              f"{os.environ.get('SFX_GEMM_TILES_PER_CTA', 'auto')}: {t * 1e3:.1f} ms {tf:.2f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
