#!/usr/bin/env python
"""Tiled Cholesky timeline from the runtime's CUDA-event trace.

    python tools/chol_timeline.py --n 32768 --b 1024 [--reps 2]

Per task kind: launch groups, summed device time (unique group intervals) and
mean; per panel step k: when POTRF(k) started / ended relative to the start of
the factorization and how long the panel chain POTRF(k) -> TRSM(k+1,k) -> the
update of A(k+1,k+1) took.  The gaps between consecutive POTRF starts are the
panel-step times; steps where they exceed the trailing-matrix work are
critical-path bound.
"""
from __future__ import annotations

import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2308_15964_b200 as sf  # noqa: E402
from paper_2308_15964_b200 import algorithms as alg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--b", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--streams", type=int, default=16)
    ap.add_argument("--every", type=int, default=1)
    a = ap.parse_args()
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, a.streams), scheduler="prio", trace=True)
    M = alg.TiledMatrix(a.n, a.b, lower=True)
    for rep in range(a.reps):
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_fill_spd(g, M, 3)
        g.wait_all()
        g2 = sf.TaskGraph().compute_on(eng)
        alg.insert_cholesky(g2, M)
        g2.wait_all()
    ev = g2.trace.export_events()
    start, end = {}, {}
    for kind, t, w, tid, _ in ev:
        if kind == "TaskStart":
            start[tid] = (t, w)
        elif kind == "TaskEnd":
            end[tid] = t
    groups = {}
    for tid, (t0, w) in start.items():
        key = (t0, end[tid], w)
        groups.setdefault(key, []).append(g2._label(tid))
    t_first = min(k[0] for k in groups)
    t_last = max(k[1] for k in groups)
    per = collections.defaultdict(lambda: [0, 0, 0.0])
    for (t0, t1, w), names in groups.items():
        nm = names[0]
        per[nm][0] += 1
        per[nm][1] += len(names)
        per[nm][2] += (t1 - t0) / 1e3
    span = (t_last - t_first) / 1e3
    print(f"makespan {span / 1e3:.2f} ms, {alg.flops_cholesky(a.n) / (span * 1e-6) / 1e12:.2f} TFLOP/s")
    print("| kind | groups | tasks | sum us | mean us |\n|---|---|---|---|---|")
    for nm, (c, nt_, s) in sorted(per.items(), key=lambda kv: -kv[1][2]):
        print(f"| {nm} | {c} | {nt_} | {s:.0f} | {s / c:.1f} |")
    # panel chain
    pot = sorted((t0, t1) for (t0, t1, w), names in groups.items() if names[0] == "potrf")
    print("\n| k | potrf start ms | potrf us | gap to next potrf start us |\n|---|---|---|---|")
    for k, (t0, t1) in enumerate(pot):
        nxt = pot[k + 1][0] if k + 1 < len(pot) else t_last
        if k % a.every == 0 or k >= len(pot) - 4:
            print(f"| {k} | {(t0 - t_first) / 1e6:.2f} | {(t1 - t0) / 1e3:.0f} | {(nxt - t0) / 1e3:.0f} |")
    eng.stop()


if __name__ == "__main__":
    main()
