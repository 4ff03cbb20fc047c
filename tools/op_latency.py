#!/usr/bin/env python
"""Latency of single tile ops (the Cholesky critical path), CUDA-event timed.

    python tools/op_latency.py [--b 1024]

Each op runs alone on an idle GPU (one task per graph, wait between reps):
POTRF(b) for b in 64..b, TRSM with inverse blocks (b x b), SYRK, NT GEMM.
"""
from __future__ import annotations

import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2308_15964_b200 as sf  # noqa: E402
from oracle import inputs  # noqa: E402


def timed(eng, build, reps=5):
    ts = []
    for r in range(reps + 1):
        g = sf.TaskGraph().compute_on(eng)
        pre = build(g)
        g.wait_all()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pre()
        g.wait_all()
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=1024)
    a = ap.parse_args()
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 4), scheduler="prio", trace=False)
    b = a.b
    for n in (64, 128, 256, 512, 1024):
        if n > b:
            break
        A0 = inputs.spd_tile(51, 0, 0, n, n, n)
        A = sf.pinned_empty((n, n))

        def build(g, A=A, A0=A0):
            A[...] = A0
            g.task(sf.write(A), device=sf.ops.potrf_inv)  # stage + factor once (warm)
            g.wait_all()

            def run():
                g.task(sf.write(A), device=sf.ops.potrf_inv)
            return run
        print(f"potrf_inv n={n}: {timed(eng, build):.1f} us")
        if n >= 128:
            def buildf(g, A=A, A0=A0):
                A[...] = A0
                g.task(sf.write(A), device=sf.ops.potrf_fullinv)
                g.wait_all()
                return lambda: g.task(sf.write(A), device=sf.ops.potrf_fullinv)
            print(f"potrf_fullinv n={n}: {timed(eng, buildf):.1f} us")
    L0 = inputs.spd_tile(51, 0, 0, b, b, b)
    L = sf.pinned_empty((b, b))
    X = sf.pinned_empty((b, b))
    C = sf.pinned_empty((b, b))
    L[...] = L0
    X[...] = inputs.uniform_tile(52, 0, 0, b, b, b)
    C[...] = inputs.uniform_tile(53, 0, 0, b, b, b)
    g0 = sf.TaskGraph().compute_on(eng)
    g0.task(sf.write(L), device=sf.ops.potrf_fullinv)
    g0.wait_all()
    cases = {
        "trsm_inv": lambda g: g.task(sf.read(L), sf.write(X), device=sf.ops.trsm_inv),
        "trsm_fullinv": lambda g: g.task(sf.read(L), sf.write(X), device=sf.ops.trsm_fullinv),
        "syrk_sub": lambda g: g.task(sf.read(X), sf.write(C), device=sf.ops.syrk_sub),
        "gemm_nt_sub": lambda g: g.task(sf.read(X), sf.read(L), sf.write(C), device=sf.ops.gemm_nt_sub),
    }
    for name, fn in cases.items():
        def build(g, fn=fn):
            fn(g)
            g.wait_all()
            return lambda: fn(g)
        print(f"{name} b={b}: {timed(eng, build):.1f} us")
    eng.stop()


if __name__ == "__main__":
    main()
