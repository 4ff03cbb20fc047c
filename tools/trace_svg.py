#!/usr/bin/env python
"""Timeline SVG + idle metric of a real CUDA run (reference trace.py:195-302).

    python tools/trace_svg.py --n 16384 --b 1024 --devices 1 --out profiles/r2_trace_chol16k.svg

Runs one tiled Cholesky with tracing on (CUDA start/end events per launch
group), writes the SVG (one lane per GPU stream, ready-count curve beneath)
and prints the per-lane and per-GPU idle metric; --ordinals 0,0 maps two
logical devices onto one GPU.
"""
import argparse
import io
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_15964_b200 as sf  # noqa: E402
from paper_2308_15964_b200 import algorithms as alg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--b", type=int, default=1024)
    ap.add_argument("--ordinals", default="0")
    ap.add_argument("--streams", type=int, default=16)
    ap.add_argument("--out", default="gpurun_out/trace.svg")
    a = ap.parse_args()
    ords = [int(x) for x in a.ordinals.split(",")]
    eng = sf.create_engine(sf.WorkerTeam.of_devices(len(ords), a.streams), scheduler="prio", trace=True,
                           ordinals=ords, group_max=8)
    M = alg.TiledMatrix(a.n, a.b, lower=True)
    g = sf.TaskGraph(trace=False).compute_on(eng)
    if len(ords) > 1:
        alg.block_cyclic(g, M, *alg.grid_shape(len(ords)))
    alg.insert_fill_spd(g, M, 3)
    g.wait_all()
    g.set_trace(True)  # the timeline shows the factorization only
    alg.insert_cholesky(g, M)
    g.wait_all()
    buf = io.StringIO()
    svg = g.generate_trace_svg(a.out, out=buf)
    print(buf.getvalue())
    rep = __import__("paper_2308_15964_b200.trace", fromlist=["idle_report"]).idle_report(g)
    print(f"span {rep['span_ms']:.3f} ms, {len(svg)} bytes of SVG -> {a.out}; violations {eng.violations()}")
    eng.stop()


if __name__ == "__main__":
    main()
