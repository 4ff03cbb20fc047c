#!/usr/bin/env python
"""Where the C2 end-to-end step loses time: the DGEMM kernels' busy fraction over
the step, from CUDA-event stamps taken AFTER each launch group's copies (runtime
option kernel_only_start), in bins.

    python tools/e2e_timeline.py [--bin-ms 5]

Same insertion as bench.py's e2e leg (insert_gemm with the wavefront skew, then
write-mode flushes of C, A, B), on the same graph across steps; the second step
is analysed.  Tracing costs some host time: the shape matters, not the total.
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
    ap.add_argument("--bin-ms", type=float, default=5.0)
    ap.add_argument("--skew", type=int, default=-1, help="insert_gemm skew (-1: 2*nt as bench.py)")
    ap.add_argument("--gps", type=int, default=4)
    ap.add_argument("--streams", type=int, default=32)
    ap.add_argument("--stage-stream", type=int, default=0)
    ap.add_argument("--stage-window", type=int, default=0, help="MiB")
    ap.add_argument("--tile-block", type=int, default=0)
    ap.add_argument("--flush-priority", type=int, default=0)
    ap.add_argument("--tail-ms", type=int, default=0)
    ap.add_argument("--skew-block", type=int, default=0)
    a = ap.parse_args()
    nt = a.n // a.b
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, a.streams), scheduler="prio", trace=True)
    eng.set_option("groups_per_stream", a.gps)
    eng.set_option("kernel_only_start", 1)
    eng.set_option("stage_stream", a.stage_stream)
    eng.set_option("flush_priority", a.flush_priority)
    eng.set_option("stage_window", a.stage_window << 20)
    A, B, C = (alg.TiledMatrix(a.n, a.b) for _ in range(3))
    g = sf.TaskGraph(trace=False).compute_on(eng)
    alg.insert_fill_uniform(g, A, 1)
    alg.insert_fill_uniform(g, B, 2)
    alg.insert_zero(g, C)
    g.wait_all()

    def step():
        if a.tile_block:
            alg.insert_gemm(g, A, B, C, tile_block=a.tile_block)
        else:
            alg.insert_gemm(g, A, B, C, skew=2 * nt if a.skew < 0 else a.skew, skew_block=a.skew_block)
        for M in (C, A, B):
            for t in M.tiles.values():
                g.flush_to_host(t)
        g.wait_all()

    step()
    g.set_trace(True)
    t0 = time.perf_counter_ns()
    step()
    t1 = time.perf_counter_ns()
    ev = g.trace.export_events()
    g0 = g._t0
    iv = {}
    for kind, t, _, tid, _ in ev:
        if kind in ("TaskStart", "TaskEnd"):
            iv.setdefault(tid, [None, None])[0 if kind == "TaskStart" else 1] = t + g0
    spans = sorted((s, e) for s, e in iv.values() if s and e and e > s)
    lo = t0
    hi = t1
    nb = int((hi - lo) / (a.bin_ms * 1e6)) + 1
    busy = [0.0] * nb
    # union of intervals, then distributed over bins
    merged = []
    for s, e in spans:
        if merged and s <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], e)
        else:
            merged.append([s, e])
    for s, e in merged:
        s = max(s, lo)
        while s < e:
            b = int((s - lo) / (a.bin_ms * 1e6))
            if b >= nb:
                break
            be = lo + (b + 1) * a.bin_ms * 1e6
            seg = min(e, be) - s
            busy[b] += seg
            s += seg
    tot_busy = sum(e - s for s, e in merged)
    st = eng.stats(0)
    print(f"h2d {st['bytes_to_device'] / 2**30:.1f} GiB, prefetches {st['prefetches']}")
    print(f"step {(hi - lo) / 1e6:.1f} ms (host clock, tracing on), kernels busy {tot_busy / 1e6:.1f} ms "
          f"({100 * tot_busy / (hi - lo):.1f} %), first kernel start +{(merged[0][0] - lo) / 1e6:.2f} ms, "
          f"last kernel end +{(merged[-1][1] - lo) / 1e6:.2f} ms of {(hi - lo) / 1e6:.1f}")
    line = []
    for b, v in enumerate(busy):
        line.append(f"{100 * v / (a.bin_ms * 1e6):3.0f}")
    for i in range(0, len(line), 20):
        print(f"  {i * a.bin_ms:6.0f} ms: " + " ".join(line[i:i + 20]))
    if a.tail_ms:
        # the last tail_ms of the step in 1 ms bins: busy % per task kind (union of
        # that kind's intervals) -- flush intervals are the D2H copies of C
        kinds = {}
        for tid, (s0, e0) in iv.items():
            if s0 and e0 and e0 > s0:
                kinds.setdefault(g._label(tid), []).append((s0, e0))
        t_lo = hi - a.tail_ms * 1e6
        for name, sp in sorted(kinds.items()):
            bins = [0.0] * int(a.tail_ms)
            cnt = [0] * int(a.tail_ms)
            for s0, e0 in sp:
                if e0 <= t_lo:
                    continue
                b0 = int(max(0, (s0 - t_lo) / 1e6))
                if b0 < len(cnt):
                    cnt[b0] += 1
            merged2 = []
            for s0, e0 in sorted(sp):
                if merged2 and s0 <= merged2[-1][1]:
                    merged2[-1][1] = max(merged2[-1][1], e0)
                else:
                    merged2.append([s0, e0])
            for s0, e0 in merged2:
                s0 = max(s0, t_lo)
                while s0 < e0:
                    bb = int((s0 - t_lo) / 1e6)
                    if bb >= len(bins):
                        break
                    be = t_lo + (bb + 1) * 1e6
                    seg = min(e0, be) - s0
                    bins[bb] += seg
                    s0 += seg
            print(f"  tail {name:6s} busy%: " + " ".join(f"{100 * v / 1e6:3.0f}" for v in bins))
            print(f"  tail {name:6s} starts: " + " ".join(f"{c:3d}" for c in cnt))
    eng.stop()


if __name__ == "__main__":
    main()
