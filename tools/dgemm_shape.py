#!/usr/bin/env python
"""One DGEMM task of an arbitrary shape, CUDA-event timed (kernel efficiency probe).

    python tools/dgemm_shape.py --m 18944 --n 128 --k 4096   # 148 tiles = one wave, long mainloop
"""
from __future__ import annotations

import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2308_15964_b200 as sf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=18944)
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--trans-b", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    peak, _ = sf.fp64_peak(0)
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 1), trace=False, device_memory=8 << 30)
    A = sf.pinned_empty((a.m, a.k))
    B = sf.pinned_empty((a.n, a.k) if a.trans_b else (a.k, a.n))
    C = sf.pinned_empty((a.m, a.n))
    g = sf.TaskGraph().compute_on(eng)
    g.task(sf.write(A), device=sf.ops.fill_uniform(1, 0, 0, a.k))
    g.task(sf.write(B), device=sf.ops.fill_uniform(2, 0, 0, B.shape[1]))
    g.task(sf.write(C), device=sf.ops.zero())
    g.wait_all()
    op = sf.ops.dgemm(1.0, 1.0, a.trans_b)
    ts = []
    for r in range(a.reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.task(sf.read(A), sf.read(B), sf.write(C), device=op)
        g.wait_all()
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1) * 1e-3)
    t = statistics.median(ts)
    fl = 2.0 * a.m * a.n * a.k
    print(f"M={a.m} N={a.n} K={a.k} trans_b={a.trans_b}: {t * 1e6:.1f} us (incl. task overhead) "
          f"{fl / t / 1e12:.2f} TFLOP/s = {fl / t / 1e12 / peak:.3f} of the DMMA peak {peak:.2f}")
    eng.stop()


if __name__ == "__main__":
    main()
