#!/usr/bin/env python
"""C3 on one GPU: kernel busy fraction over one factorization (launch groups'
CUDA-event intervals, start stamped after each group's copies), in bins, and
the time per op class (union of that class's intervals).

    python tools/chol_busy.py [--n 32768 --b 1024 --bin-ms 10]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_15964_b200 as sf  # noqa: E402
from paper_2308_15964_b200 import algorithms as alg  # noqa: E402


def union(spans):
    m = []
    for s, e in sorted(spans):
        if m and s <= m[-1][1]:
            m[-1][1] = max(m[-1][1], e)
        else:
            m.append([s, e])
    return m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--b", type=int, default=1024)
    ap.add_argument("--bin-ms", type=float, default=10.0)
    a = ap.parse_args()
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 32), scheduler="prio", trace=True, group_max=8)
    eng.set_option("kernel_only_start", 1)
    M = alg.TiledMatrix(a.n, a.b, lower=True)
    g = sf.TaskGraph(trace=False).compute_on(eng)
    for rep in range(2):
        alg.insert_fill_spd(g, M, 3)
        g.wait_all()
        if rep == 1:
            g.set_trace(True)
        t0 = time.perf_counter_ns()
        alg.insert_cholesky(g, M)
        g.wait_all()
        t1 = time.perf_counter_ns()
    names = dict(g._names)
    for first, n, rn in g._name_ranges:
        for k in range(n):
            names[first + k] = rn[k] if isinstance(rn, (list, tuple)) else rn
    iv = {}
    for kind, t, _, tid, _ in g.trace.export_events():
        if kind in ("TaskStart", "TaskEnd"):
            iv.setdefault(tid, [None, None])[0 if kind == "TaskStart" else 1] = t + g._t0
    spans = [(s, e, names.get(tid, "?")) for tid, (s, e) in iv.items() if s and e and e > s]
    allm = union([(s, e) for s, e, _ in spans])
    busy = sum(e - s for s, e in allm)
    print(f"factorization {(t1 - t0) / 1e6:.1f} ms (host clock, tracing on), kernels busy {busy / 1e6:.1f} ms "
          f"({100 * busy / (t1 - t0):.1f} %)")
    for cls in sorted({n for _, _, n in spans}):
        m = union([(s, e) for s, e, n in spans if n == cls])
        print(f"  {cls:12s} union {sum(e - s for s, e in m) / 1e6:7.1f} ms, {sum(1 for _, _, n in spans if n == cls)} tasks")
    nb = int((t1 - t0) / (a.bin_ms * 1e6)) + 1
    bins = [0.0] * nb
    for s, e in allm:
        s = max(s, t0)
        while s < e:
            b = int((s - t0) / (a.bin_ms * 1e6))
            if b >= nb:
                break
            be = t0 + (b + 1) * a.bin_ms * 1e6
            seg = min(e, be) - s
            bins[b] += seg
            s += seg
    line = [f"{100 * v / (a.bin_ms * 1e6):3.0f}" for v in bins]
    for i in range(0, len(line), 20):
        print(f"  {i * a.bin_ms:6.0f} ms: " + " ".join(line[i:i + 20]))
    eng.stop()


if __name__ == "__main__":
    main()
