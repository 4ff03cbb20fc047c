#!/usr/bin/env python
"""Kernel time and accuracy of the panel-chain ops alone on an idle B200.

    python tools/potrf_probe.py [--sizes 256,512,1024,2048] [--reps 5]
    SFX_POTRF=coop python tools/potrf_probe.py      (round-1 cooperative POTRF, A/B)

Every rep regenerates the input on the device (fill_spd / fill_uniform ops), then
runs ONE op; its launch group's CUDA-event time (engine kernel_timing) is the
number.  Checks: ||A - L L^T|| / ||A||, and for the inverse modes the stored
inverse blocks (upper triangle) against inv(L); TRSM: ||X L^T - B|| / ||B||.
"""
from __future__ import annotations

import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2308_15964_b200 as sf  # noqa: E402
from oracle import inputs  # noqa: E402


def op_time(eng, g, prep, run, reps):
    ts = []
    for _ in range(reps + 1):
        prep()
        g.wait_all()
        t0 = eng.stats(0)["timed_ns"]
        run()
        g.wait_all()
        ts.append((eng.stats(0)["timed_ns"] - t0) / 1e3)
    return statistics.median(ts[1:]), min(ts[1:])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="256,512,1024,2048")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 4), scheduler="prio", trace=False, kernel_timing=True)
    g = sf.TaskGraph().compute_on(eng)
    for n in [int(x) for x in a.sizes.split(",")]:
        A0 = inputs.spd_tile(51, 0, 0, n, n, n)
        A = sf.pinned_empty((n, n))
        for name, op in (("potrf", sf.ops.potrf), ("potrf_inv", sf.ops.potrf_inv),
                         ("potrf_fullinv", sf.ops.potrf_fullinv)):
            med, best = op_time(eng, g, lambda: g.task(sf.write(A), device=sf.ops.fill_spd(51, 0, 0, n)),
                                lambda: g.task(sf.write(A), device=op), a.reps)
            g.flush_to_host(A, keep_device=True)
            g.wait_all()
            L = np.tril(A)
            res = np.linalg.norm(A0 - L @ L.T) / np.linalg.norm(A0)
            extra = ""
            if name == "potrf":
                extra = f" upper untouched {np.array_equal(np.triu(A, 1), np.triu(A0, 1))}"
            elif name == "potrf_inv":
                worst = 0.0
                for k in range(0, n, 64):
                    Lk = L[k:k + 64, k:k + 64]
                    W = np.triu(A[k:k + 64, k:k + 64], 1).T + np.diag(1.0 / np.diag(Lk))
                    worst = max(worst, np.abs(W @ Lk - np.eye(64)).max())
                extra = f" max|inv(L_kk) L_kk - I| {worst:.2e}"
            else:
                W = np.triu(A, 1).T + np.diag(1.0 / np.diag(L))
                extra = f" max|W L - I| {np.abs(W @ L - np.eye(n)).max():.2e}"
            flops = n ** 3 / 3 * (2 if name == "potrf_fullinv" else 1)
            print(f"{name} n={n}: {med:.1f} us (best {best:.1f}), {flops / med / 1e6:.2f} TFLOP/s, "
                  f"residual {res:.2e}{extra}", flush=True)
        # TRSM with the full inverse (L from the last potrf_fullinv)
        B = sf.pinned_empty((n, n))
        B0 = inputs.uniform_tile(52, 0, 0, n, n, n)
        med, best = op_time(eng, g, lambda: g.task(sf.write(B), device=sf.ops.fill_uniform(52, 0, 0, n)),
                            lambda: g.task(sf.read(A), sf.write(B), device=sf.ops.trsm_fullinv), a.reps)
        g.flush_to_host(B, keep_device=True)
        g.wait_all()
        L = np.tril(A)
        res = np.linalg.norm(B @ L.T - B0) / np.linalg.norm(B0)
        print(f"trsm_fullinv n={n}: {med:.1f} us (best {best:.1f}), {n ** 3 / med / 1e6:.2f} TFLOP/s, "
              f"residual {res:.2e}", flush=True)
        # the other two panel-chain ops, alone: SYRK (lower) and the NT GEMM update
        C = sf.pinned_empty((n, n))
        med, best = op_time(eng, g, lambda: g.task(sf.write(C), device=sf.ops.fill_spd(53, 0, 0, n)),
                            lambda: g.task(sf.read(B), sf.write(C), device=sf.ops.syrk_sub), a.reps)
        print(f"syrk_sub n={n}: {med:.1f} us (best {best:.1f}), {n ** 3 / med / 1e6:.2f} TFLOP/s", flush=True)
        med, best = op_time(eng, g, lambda: g.task(sf.write(C), device=sf.ops.fill_spd(53, 0, 0, n)),
                            lambda: g.task(sf.read(B), sf.read(A), sf.write(C), device=sf.ops.gemm_nt_sub), a.reps)
        print(f"gemm_nt_sub n={n}: {med:.1f} us (best {best:.1f}), {2 * n ** 3 / med / 1e6:.2f} TFLOP/s", flush=True)
    eng.stop()


if __name__ == "__main__":
    main()
