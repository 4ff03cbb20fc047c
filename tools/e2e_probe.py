#!/usr/bin/env python
"""Host<->device transfer ceilings and the e2e GEMM step's transfer/compute overlap.

    python tools/e2e_probe.py [--n 16384 --b 512]

1. pinned H2D, D2H and simultaneous H2D+D2H bandwidth (torch copies, 1 GiB);
2. e2e C2 steps (host tiles -> device -> host, as bench.py's e2e leg) under the
   given runtime knobs (prefetch on/off and depth, streams, groups per stream).
"""
from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2308_15964_b200 as sf  # noqa: E402
from paper_2308_15964_b200 import algorithms as alg  # noqa: E402


def bw():
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name in ("h2d", "d2h", "both"):
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if name in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d.copy_(h, non_blocking=True)
            if name in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        out[name] = (n * (2 if name == "both" else 1)) / dt / 1e9
    print({k: round(v, 1) for k, v in out.items()}, "GB/s (both = sum of the two directions)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--b", type=int, default=512)
    ap.add_argument("--streams", type=int, default=16)
    ap.add_argument("--prefetch", type=int, default=1)
    ap.add_argument("--depth", type=int, default=64)
    ap.add_argument("--gps", type=int, default=2)
    ap.add_argument("--no-bw", action="store_true")
    ap.add_argument("--row-block", type=int, default=0, help="insert_gemm priorities (row-block height, 0 = off)")
    ap.add_argument("--tile-block", type=int, default=0, help="insert_gemm tile_block (h x h C blocks, 0 = off)")
    ap.add_argument("--skew", type=int, default=0, help="insert_gemm skew (wavefront over S waves, 0 = off)")
    a = ap.parse_args()
    if not a.no_bw:
        bw()
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, a.streams), scheduler="prio", trace=False)
    eng.set_option("prefetch", a.prefetch)
    eng.set_option("prefetch_depth", a.depth)
    eng.set_option("groups_per_stream", a.gps)
    print(vars(a))
    A, B, C = (alg.TiledMatrix(a.n, a.b) for _ in range(3))
    g = sf.TaskGraph().compute_on(eng)
    alg.insert_fill_uniform(g, A, 1)
    alg.insert_fill_uniform(g, B, 2)
    alg.insert_zero(g, C)
    g.wait_all()

    def e2e_step(gr):
        alg.insert_gemm(gr, A, B, C, priorities=a.row_block, tile_block=a.tile_block, skew=a.skew)
        for M in (C, A, B):
            for t in M.tiles.values():
                gr.flush_to_host(t)
        gr.wait_all()

    e2e_step(g)
    for rep in range(2):
        g2 = sf.TaskGraph().compute_on(eng)
        s0 = eng.stats(0)
        t0 = time.perf_counter()
        e2e_step(g2)
        dt = time.perf_counter() - t0
        s1 = eng.stats(0)
        print(f"e2e step {dt * 1e3:.1f} ms  {alg.flops_gemm(a.n) / dt / 1e12:.2f} TFLOP/s  "
              f"H2D {(s1['bytes_to_device'] - s0['bytes_to_device']) / 1e9:.2f} GB  "
              f"D2H {(s1['bytes_from_device'] - s0['bytes_from_device']) / 1e9:.2f} GB  "
              f"prefetches {s1['prefetches'] - s0['prefetches']}")
    eng.stop()


if __name__ == "__main__":
    main()
