"""Per-step C2 times after a long back-to-back insertion burst in the same graph
(DESIGN §6c open issue): K pipelined steps, then isolated steps one by one with
the runtime's host counters per step.

    python tools/burst_probe.py [K] [after]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2308_15964_b200 as sf  # noqa: E402
from paper_2308_15964_b200 import algorithms as alg  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
after = int(sys.argv[2]) if len(sys.argv) > 2 else 6
n, b = 16384, 512
eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 32), scheduler="prio", trace=False, group_max=32)
A, B, C = (alg.TiledMatrix(n, b) for _ in range(3))
g = sf.TaskGraph().compute_on(eng)
alg.insert_fill_uniform(g, A, 1)
alg.insert_fill_uniform(g, B, 2)
alg.insert_zero(g, C)
g.wait_all()
flops = alg.flops_gemm(n)


def timed(fn):
    s0 = eng.stats(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record()
    ins = fn()
    e1.record()
    torch.cuda.synchronize()
    s1 = eng.stats(0)
    t = e0.elapsed_time(e1) / 1e3
    nt = max(1, s1["tasks_executed"] - s0["tasks_executed"])
    per = {k: round((s1[k] - s0[k]) / 1e3 / nt, 3) for k in ("t_plan_ns", "t_issue_ns", "t_complete_ns")}
    return t, ins, per, time.perf_counter() - h0


def one():
    t0 = time.perf_counter()
    alg.insert_gemm(g, A, B, C)
    ins = time.perf_counter() - t0
    g.wait_all()
    return ins


for i in range(3):
    t, ins, per, _ = timed(one)
    print(f"before  step {i}: {flops / t / 1e12:.2f} TFLOP/s  insert {ins * 1e3:.1f} ms  {per}", flush=True)


def burst():
    t0 = time.perf_counter()
    for _ in range(K):
        alg.insert_gemm(g, A, B, C)
    ins = time.perf_counter() - t0
    g.wait_all()
    return ins


t, ins, per, _ = timed(burst)
print(f"burst x{K}: {K * flops / t / 1e12:.2f} TFLOP/s  insert {ins * 1e3:.1f} ms  {per}", flush=True)
for i in range(after):
    t, ins, per, _ = timed(one)
    print(f"after   step {i}: {flops / t / 1e12:.2f} TFLOP/s  insert {ins * 1e3:.1f} ms  {per}", flush=True)
eng.stop()
