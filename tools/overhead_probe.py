"""The reference overhead protocol (bench.overhead_gpu) on the GPU engine for a
few configurations, plus where the host time goes (per-task executor plan /
issue / release and completion-thread time from the runtime's own counters).

    python tools/overhead_probe.py [T] [N]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2308_15964_b200 as sf  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else (os.cpu_count() or 4)
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
for D, mode, deps in ((0.0, "write", 1), (0.0, "commute", 1), (1e-4, "write", 1), (1e-3, "write", 1),
                      (1e-3, "commute", 1), (1e-4, "write", 20)):
    r = bench.overhead_gpu(sf, 0, T, N, D, mode, deps, reps=2)
    print(f"D={D:g} {mode} deps={deps}: " + " ".join(f"{k}={v:.2f}" for k, v in r.items()), flush=True)

# host-side cost breakdown at D = 0 (trace on, as in the protocol, and off)
for trace in (True, False):
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, T), trace=trace, device_memory=1 << 26)
    g = sf.TaskGraph().compute_on(eng)
    cells = [sf.Cell(0) for _ in range(T)]
    for c in cells:
        g.task(sf.write(c), device=sf.ops.noop)
    g.wait_all()
    s0 = eng.stats(0)
    t0 = time.perf_counter_ns()
    for i in range(N):
        for c in cells:
            g.task(sf.write(c), device=sf.ops.noop)
    t_ins = time.perf_counter_ns() - t0
    g.wait_all()
    t_all = time.perf_counter_ns() - t0
    s1 = eng.stats(0)
    n = T * N
    d = {k: (s1[k] - s0[k]) / n / 1e3 for k in ("t_plan_ns", "t_issue_ns", "t_release_ns", "t_complete_ns")}
    print(f"trace={trace}: insert {t_ins / n / 1e3:.2f} us/task, total {t_all / n / 1e3:.2f} us/task, groups "
          f"{(s1['groups'] - s0['groups']) / n:.2f}/task, per task: "
          + " ".join(f"{k}={v:.2f}us" for k, v in d.items()), flush=True)
    eng.stop()
