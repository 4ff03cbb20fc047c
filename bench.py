#!/usr/bin/env python
"""Benchmark of the STF GPU execution path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one process per GPU)

Workload at N=1 (BASELINE.json configs[1]): tiled DGEMM 16384 x 16384 FP64
with 512 x 512 tiles ("1024 tiles") -> 32,768 GEMM tasks per step, inserted
through the drop-in TaskGraph API and executed by the native runtime.  A step
is one full tiled C += A B pass; inputs (3 x 2 GiB) are far larger than the
126 MB L2, so no flush is needed between steps.  With N ranks every rank runs
its own C2 instance on its GPU (weak scaling, no data-path collective: the
DGEMM configs are 1 GPU per config).

Legs of the JSON line:
  value      device-resident inputs, FP64 GFLOP/s summed over ranks (CUDA
             events on the device, max step time over ranks)
  e2e        same metric through the public API from pinned HOST buffers: every
             step stages A, B, C host->device on demand and flushes C back
  roofline   FP64 DMMA pipe: achieved TFLOP/s of the DGEMM kernel over the timed
             region vs the DMMA peak measured in-run on this GPU
  cpu_baseline  the reference algorithm on the host cores (oracle restatement of
             the reference STF engine + numpy bodies; rank 0, N=1), bounded sample
  secondary  Cholesky 32768/1024 (C3) and particles 2^20/256 groups (C4) on one
             GPU, and the runtime overhead in us/task (reference protocol)
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 GFLOP/s tiled Cholesky/GEMM at 1/2/4/8 B200 (% FP64 peak); µs/task"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=("gemm", "cholesky", "particles"), default="gemm",
                    help="gemm: C2 tiled DGEMM (default, BASELINE configs[1]); cholesky: tiled Cholesky over "
                         "all --gpus GPUs from one runtime (C3 at n=32768/1024, C5 at n=65536/1024); "
                         "particles: C4 (2^20 particles, 256 groups) over all --gpus GPUs from one runtime")
    ap.add_argument("--n", "--matrix-n", dest="n", type=int, default=None)
    ap.add_argument("--b", "--tile-b", dest="b", type=int, default=None)
    ap.add_argument("--streams", type=int, default=32)
    ap.add_argument("--group", type=int, default=32)
    ap.add_argument("--chol-group", type=int, default=8,
                    help="launch-group size for the Cholesky legs (tools/chol_sweep.py: 8 best for b=1024)")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--e2e-row-priorities", type=int, default=0)
    ap.add_argument("--e2e-skew", type=int, default=-1, help="insert_gemm skew on the e2e leg (-1: 2*nt, 0: FIFO)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


# ----------------------------------------------------------------- distributed

class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.backend = None

    def init(self, backend="nccl"):
        self.backend = backend
        if self.world > 1:
            import torch
            import torch.distributed as dist

            if backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device="cuda" if self.backend == "nccl" else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def done(self):
        if self.pg:
            self.pg.destroy_process_group()


# ----------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._th = threading.Thread(target=run, daemon=True)
        self._th.start()

    def stop(self):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            for name, v in zip(names, s[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------- CPU leg

def cpu_baseline(n: int, b: int, seconds: float, steps: int = 1, warmup: int = 0):
    """Reference algorithm on the host: the oracle's restatement of the reference
    STF engine (one worker thread per core) running numpy tile bodies, on the
    first block-rows of the same tiled DGEMM (bounded sample).  One calibration
    pass sizes the sample to about `seconds`; then `warmup` untimed and `steps`
    timed samples run, and the mean rate of the timed ones is returned."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import bodies, stf

    cores = os.cpu_count() or 1
    nt = n // b
    rng = np.random.default_rng(1)
    A = [[rng.random((b, b)) for _ in range(nt)] for _ in range(2)]
    B = [[rng.random((b, b)) for _ in range(nt)] for _ in range(nt)]

    def run_rows(rows):
        C = [[np.zeros((b, b)) for _ in range(nt)] for _ in range(rows)]
        orc = stf.Oracle(workers=cores, trace=False)
        t0 = time.perf_counter()
        for i in range(rows):
            for j in range(nt):
                for k in range(nt):
                    orc.task([(stf.READ, A[i % 2][k]), (stf.READ, B[k][j]), (stf.WRITE, C[i][j])],
                             body=bodies.gemm_nn)
        orc.wait_all()
        dt = time.perf_counter() - t0
        orc.stop()
        return dt

    with threadpool_limits(1):
        t1 = run_rows(1)
        rows = max(1, min(nt, int(seconds / max(t1, 1e-3))))
        for _ in range(warmup):
            run_rows(rows)
        dts = [run_rows(rows) for _ in range(max(1, steps))]
    dt = statistics.mean(dts)
    flops = 2.0 * b ** 3 * nt * nt * rows
    # library ceiling for context: one monolithic multithreaded
    # OpenBLAS product of 4096^2 FP64 with every host thread
    m = 4096
    X, Y = rng.random((m, m)), rng.random((m, m))
    X @ Y
    t0 = time.perf_counter()
    X @ Y
    lib = 2.0 * m ** 3 / (time.perf_counter() - t0) / 1e9
    return {"value": flops / dt / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "port",
            "library_ceiling_gflops": lib, "library_ceiling": f"numpy/OpenBLAS {m}^2 FP64 A@B, all host threads",
            "sample": f"tiled DGEMM {n}/{b}: block-rows 0..{rows - 1} of C ({rows * nt * nt} tasks, "
                      f"{flops / 1e12:.2f} TFLOP per sample) on the oracle STF engine (restated reference, "
                      f"{cores} host worker threads, numpy bodies, 1 BLAS thread each); "
                      f"{len(dts)} timed sample(s), mean",
            "seconds": dt}


def run_reference(args, dist):
    if dist.rank != 0:
        return  # under torchrun only rank 0 runs the CPU reference
    args.n, args.b = args.n or 16384, args.b or 512
    # each step is a bounded sample; the whole --steps/--warmup run stays within a few minutes
    per_step = max(1.0, min(args.cpu_seconds, 150.0 / max(1, args.steps + args.warmup)))
    res = cpu_baseline(args.n, args.b, per_step, steps=args.steps, warmup=args.warmup)
    nt = args.n // args.b
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["seconds"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"tiled DGEMM {args.n}x{args.n} fp64, {args.b}x{args.b} tiles (BASELINE configs[1], "
                               f"C2), {nt ** 3} GEMM tasks per step per GPU",
                   "n": args.n, "b": args.b, "cpu_sample": res["sample"]},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample",
                                             "library_ceiling_gflops", "library_ceiling")},
        "e2e": {"value": res["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU legs

def main_ours(args, dist):
    import numpy as np
    import torch

    import paper_2308_15964_b200 as sf
    from paper_2308_15964_b200 import algorithms as alg

    dev = dist.local if dist.world > 1 else 0
    torch.cuda.set_device(dev)
    peak_tf, _ = sf.fp64_peak(dev)
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, args.streams), scheduler="prio", trace=False,
                           ordinals=[dev], group_max=args.group, kernel_timing=True)
    n, b = args.n, args.b
    nt = n // b
    flops = alg.flops_gemm(n)
    A, B, C = (alg.TiledMatrix(n, b) for _ in range(3))
    g = sf.TaskGraph().compute_on(eng)
    alg.insert_fill_uniform(g, A, 1)
    alg.insert_fill_uniform(g, B, 2)
    alg.insert_zero(g, C)
    g.wait_all()

    def step():
        alg.insert_gemm(g, A, B, C)
        g.wait_all()

    if os.environ.get("SFX_BENCH_KTIME", "1") == "0":  # diagnostics: the device leg without timing events
        eng.set_option("kernel_timing", 0)

    for _ in range(args.warmup):
        step()
    st0 = eng.stats(0)
    clocks = ClockSampler(dev)
    clocks.start()
    times = []
    for _ in range(args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    clk = clocks.stop()
    st1 = eng.stats(0)
    step_s = dist.max(statistics.mean(times))
    value = flops * dist.world / step_s / 1e9
    launches = st1["kernel_launches"] - st0["kernel_launches"]

    # ---- e2e: host-resident inputs through the public API ----
    def e2e_step():
        # wavefront priorities (insert_gemm skew): the k-chains of the C tiles start
        # staggered over 2*nt waves, so C's staging (2 GiB H2D) and its flush
        # (2 GiB D2H) spread over the step instead of piling up in the first and
        # last waves (tools/e2e_probe.py: 25.7 -> 28.3 TFLOP/s)
        alg.insert_gemm(g, A, B, C, priorities=args.e2e_row_priorities,
                        skew=args.e2e_skew if args.e2e_skew >= 0 else 2 * nt)
        for t in C.tiles.values():
            g.flush_to_host(t)                      # C back to the host (write-mode flush)
        for M in (A, B):
            for t in M.tiles.values():
                g.flush_to_host(t)                  # clean copies dropped: next step restages
        g.wait_all()

    # more launch groups queued per stream keeps the copy engines and the SMs both
    # busy while tiles stream in (tools/e2e_probe.py: 22.4 -> 25.5-26 TFLOP/s)
    eng.set_option("groups_per_stream", 4)
    # the launch-group timing events serve the kernel roofline only (device leg);
    # the e2e leg runs the product configuration without them
    eng.set_option("kernel_timing", 0)
    e2e_step()  # first pass moves everything to the host side
    s0 = eng.stats(0)
    et = []
    for _ in range(max(2, args.steps // 2)):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        e2e_step()
        e1.record()
        torch.cuda.synchronize()
        et.append(e0.elapsed_time(e1) / 1e3)
    s1 = eng.stats(0)
    ksteps = len(et)
    e2e_s = dist.max(statistics.mean(et))
    e2e = {"value": flops * dist.world / e2e_s / 1e9, "unit": "GFLOP/s",
           "h2d_bytes_per_step": (s1["bytes_to_device"] - s0["bytes_to_device"]) // ksteps,
           "d2h_bytes_per_step": (s1["bytes_from_device"] - s0["bytes_from_device"]) // ksteps,
           "ms_per_step": e2e_s * 1e3}
    eng.stop()
    del A, B, C

    traffic = None
    tpath = os.path.join(ROOT, "profiles", "dgemm_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            # ncu --set full capture of one grouped launch of the same shape: scale to this run's
            # mean tasks per launch (traffic is per task: A, B tiles read, C read + written)
            traffic = tj["bytes_per_task"] * (st1["timed_tasks"] - st0["timed_tasks"]) / max(
                1, st1["timed_groups"] - st0["timed_groups"])
        except Exception:
            traffic = None
    # kernel timing: every launch group is bracketed by CUDA events recorded on the stream it is
    # launched on (runtime flag SFX_FLAG_KTIME); busy_ns is the union of those intervals (groups on
    # different streams overlap), timed_ns their sum
    groups = st1["timed_groups"] - st0["timed_groups"]
    tasks = st1["timed_tasks"] - st0["timed_tasks"]
    sum_ns = st1["timed_ns"] - st0["timed_ns"]
    busy_ns = st1["busy_ns"] - st0["busy_ns"]
    flop_task = 2.0 * b ** 3
    achieved = tasks * flop_task / (busy_ns * 1e-9) / 1e12 if busy_ns else value / dist.world / 1e3
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": achieved / peak_tf, "traffic": traffic,
                "peak_source": "FP64 DMMA (mma.sync m8n8k4 -> DMMA.8x8x4) peak measured in-run on this GPU "
                               "by sfx_fp64_peak; MEASURED_PEAKS.json has no FP64 entry",
                "kernel": "dgemm_dmma_kernel (grouped, persistent, TMA + DMMA)",
                "algorithmic_flops_per_task": flop_task,
                "launches": groups, "tasks_per_launch": tasks / max(groups, 1),
                "algorithmic_flops_per_launch": tasks * flop_task / max(groups, 1),
                "launch_avg_us": sum_ns / max(groups, 1) / 1e3,
                "launch_concurrency": sum_ns / busy_ns if busy_ns else None,
                "kernel_share_of_step": busy_ns * 1e-9 / (sum(times)) if busy_ns else None,
                "achieved_how": "algorithmic flops of the timed launches / union of their CUDA-event "
                                "intervals on the launching streams (timed region only)"}

    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": dist.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (splitmix64 uniform tiles generated on device)",
        "config": {"workload": f"tiled DGEMM {n}x{n} fp64, {b}x{b} tiles (BASELINE configs[1], C2), "
                               f"{nt ** 3} GEMM tasks per step per GPU",
                   "n": n, "b": b, "tasks_per_step": nt ** 3, "streams_per_gpu": args.streams,
                   "group_max": args.group, "scheduler": "prio",
                   "l2": "inputs (6 GiB) larger than L2; no flush", "parallelism": f"replica x{dist.world}"},
        "clocks": clk, "e2e": e2e, "gpu_launches": launches, "roofline": roofline,
        "pct_fp64_peak": 100.0 * value / dist.world / 1e3 / peak_tf,
    }

    if dist.rank == 0 and dist.world == 1 and not args.no_secondary:
        line["secondary"] = secondary(sf, alg, dev, args, peak_tf)
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu:
        try:
            cb = cpu_baseline(n, b, args.cpu_seconds)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                       "library_ceiling_gflops", "library_ceiling")}
        except Exception as exc:  # the CPU leg must not hide the GPU line
            line["cpu_baseline"] = {"error": repr(exc)}
    if dist.rank == 0:
        print(json.dumps(line), flush=True)


def secondary(sf, alg, dev, args, peak_tf):
    import torch

    out = {}
    # C3: tiled Cholesky 32768 / 1024 on one GPU
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, args.streams), scheduler="prio", trace=False,
                           ordinals=[dev], group_max=args.chol_group)
    n, b = 32768, 1024
    M = alg.TiledMatrix(n, b, lower=True)
    g = sf.TaskGraph().compute_on(eng)
    ts = []
    for rep in range(3):
        alg.insert_fill_spd(g, M, 3)
        g.wait_all()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        alg.insert_cholesky(g, M)
        g.wait_all()
        e1.record()
        torch.cuda.synchronize()
        if rep:
            ts.append(e0.elapsed_time(e1) / 1e3)
    t = statistics.mean(ts)
    out["cholesky_C3"] = {"n": n, "b": b, "tasks": 5984, "seconds": t, "gflops": alg.flops_cholesky(n) / t / 1e9,
                          "pct_fp64_peak": 100 * alg.flops_cholesky(n) / t / 1e12 / peak_tf}
    eng.stop()
    del M
    # C4: particles 2^20 in 256 groups, one evaluation
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, args.streams), trace=False, ordinals=[dev],
                           kernel_timing=True)
    ng, per = 256, 4096
    P = [sf.pinned_empty((4, per)) for _ in range(ng)]
    F = [sf.pinned_empty((4, per)) for _ in range(ng)]
    g = sf.TaskGraph().compute_on(eng)
    alg.insert_fill_particles(g, P, 4)
    for f in F:
        g.task(sf.write(f), device=sf.ops.zero())
    g.wait_all()
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        s0 = eng.stats(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        alg.insert_particles(g, P, F)
        g.wait_all()
        e1.record()
        torch.cuda.synchronize()
        s1 = eng.stats(0)
        if rep:
            ts.append(e0.elapsed_time(e1) / 1e3)
    t = statistics.mean(ts)
    inter = alg.interactions(ng * per)
    dfma_tf = sf.fp64_dfma_peak(dev)
    # mutual kernel: 23 FP64 instructions per unordered pair = 2 ordered interactions
    # (csrc/kernels/particles.cu); FP64-pipe bound = (DFMA peak / 2 flop) instr/s / 11.5
    bound = dfma_tf * 1e12 / 2 / 11.5
    busy = (s1["busy_ns"] - s0["busy_ns"]) * 1e-9
    out["particles_C4"] = {"particles": ng * per, "groups": ng, "tasks": 32896, "seconds": t,
                           "interactions_per_s": inter / t,
                           "gflops_20flop_convention": inter * alg.FLOP_PER_INTERACTION / t / 1e9,
                           "roofline": {"bound": "fp64 pipe (DFMA/DMUL/DADD)", "unit": "interactions/s",
                                        "achieved": inter / busy if busy else None,
                                        "peak": bound, "frac": inter / busy / bound if busy else None,
                                        "dfma_peak_tflops": dfma_tf,
                                        "fp64_instr_per_interaction": 11.5,
                                        "kernel_share_of_step": busy / t,
                                        "launches": s1["timed_groups"] - s0["timed_groups"]}}
    eng.stop()
    # runtime overhead per task: reference protocol (src/bench.py:67-117): T chains x N
    # tasks, each task writes (or commutatively writes) its chain cell and runs for D;
    # O_avg = makespan / N - D per chain step, insertion cost per task
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 4), trace=False, ordinals=[dev])
    T, N = 4, 2000
    rows = []
    for mode in ("write", "commute"):
        acc = sf.write if mode == "write" else sf.commutative_write
        for D in (0.0, 10e-6):
            op = sf.ops.noop if D == 0 else sf.ops.spin(int(D * 1e9))
            g = sf.TaskGraph().compute_on(eng)
            cells = [sf.Cell(0) for _ in range(T)]
            res = []
            for rep in range(3):
                t0 = time.perf_counter()
                for i in range(N):
                    for c in cells:
                        g.task(acc(c), device=op)
                t1 = time.perf_counter()
                g.wait_all()
                t2 = time.perf_counter()
                if rep:
                    res.append(((t1 - t0) / (T * N), (t2 - t0) / N - D))
            rows.append({"mode": mode, "D_us": D * 1e6, "T": T, "N": N,
                         "insert_us_per_task": 1e6 * statistics.mean(r[0] for r in res),
                         "O_avg_us": 1e6 * statistics.mean(r[1] for r in res),
                         "O_avg_us_per_task": 1e6 * statistics.mean(r[1] for r in res) / T})
    out["runtime_overhead"] = {"protocol": "reference src/bench.py:67-117: T chains x N tasks, O_avg = "
                                           "makespan/N - D (wall clock from first insertion to wait_all), "
                                           "Python per-task insertion", "runs": rows}
    eng.stop()
    return out


def main_cholesky(args, dist):
    """Tiled Cholesky over all GPUs of the node from ONE runtime (rank 0).

    The STF runtime is a single-process multi-device engine (the reference's
    WorkerTeam.of_host_and_device_workers(devices=N)); placement is owner-computes
    on a 2-D block-cyclic tile distribution and remote panels move peer-to-peer
    over NVLink.  Under torchrun, ranks > 0 only join the barriers.
    """
    import torch

    import paper_2308_15964_b200 as sf
    from paper_2308_15964_b200 import algorithms as alg

    ndev = max(args.gpus, dist.world)
    if dist.rank != 0:
        dist.barrier()
        return
    n, b = args.n or 32768, args.b or 1024
    nt = n // b
    peak_tf, _ = sf.fp64_peak(0)
    eng = sf.create_engine(sf.WorkerTeam.of_devices(ndev, args.streams), scheduler="prio", trace=False,
                           ordinals=list(range(ndev)), group_max=args.chol_group)
    M = alg.TiledMatrix(n, b, lower=True)
    P, Q = alg.grid_shape(ndev)
    times = []
    clocks = ClockSampler(0)
    for rep in range(args.warmup + args.steps):
        g = sf.TaskGraph().compute_on(eng)
        alg.block_cyclic(g, M, P, Q)
        alg.insert_fill_spd(g, M, 3)
        g.wait_all()
        for d in range(ndev):
            torch.cuda.synchronize(d)
        if rep == args.warmup:
            clocks.start()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        alg.insert_cholesky(g, M)
        g.wait_all()
        e1.record()
        torch.cuda.synchronize()
        if rep >= args.warmup:
            times.append(e0.elapsed_time(e1) / 1e3)
    clk = clocks.stop()
    stats = [eng.stats(d) for d in range(ndev)]
    eng.stop()
    t = statistics.mean(times)
    flops = alg.flops_cholesky(n)
    value = flops / t / 1e9
    ntasks = nt + nt * (nt - 1) + nt * (nt - 1) * (nt - 2) // 6  # potrf + trsm + syrk + gemm
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ndev, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic SPD (R+R^T)/2 + n*I, generated on device",
        "config": {"workload": f"tiled Cholesky {n}x{n} fp64, {b}x{b} tiles, {ndev} GPU(s) from one runtime",
                   "n": n, "b": b, "tasks": ntasks, "grid": [P, Q], "streams_per_gpu": args.streams,
                   "parallelism": f"owner-computes 2-D block-cyclic {P}x{Q}, NVLink peer pulls",
                   "l2": "working set (%.1f GiB) larger than L2" % (len(M.tiles) * b * b * 8 / 2 ** 30)},
        "clocks": clk,
        "pct_fp64_peak": 100.0 * value / 1e3 / (peak_tf * ndev),
        "roofline": {"bound": "tensor", "achieved": value / 1e3 / ndev, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": value / 1e3 / ndev / peak_tf, "traffic": None,
                     "peak_source": "FP64 DMMA peak measured in-run (sfx_fp64_peak), per GPU"},
        "p2p_bytes": sum(s["bytes_p2p_in"] for s in stats),
        "gpu_launches": stats[0]["kernel_launches"],
    }
    print(json.dumps(line), flush=True)
    dist.barrier()


def main_particles(args, dist):
    """C4 over all GPUs of the node from ONE runtime (rank 0): pair tasks dealt to the
    GPUs, per-GPU partial accumulators, one dacc reduction per group."""
    import torch

    import paper_2308_15964_b200 as sf
    from paper_2308_15964_b200 import algorithms as alg

    ndev = max(args.gpus, dist.world)
    if dist.rank != 0:
        dist.barrier()
        return
    ng, per = 256, 4096
    dfma_tf = sf.fp64_dfma_peak(0)
    eng = sf.create_engine(sf.WorkerTeam.of_devices(ndev, args.streams), trace=False, ordinals=list(range(ndev)),
                           group_max=args.group)
    P = [sf.pinned_empty((4, per)) for _ in range(ng)]
    F = [sf.pinned_empty((4, per)) for _ in range(ng)]
    g = sf.TaskGraph().compute_on(eng)
    alg.insert_fill_particles(g, P, 4)
    g.wait_all()
    parts = None
    times = []
    clocks = ClockSampler(0)
    for rep in range(args.warmup + args.steps):
        for f in F:
            g.task(sf.write(f), device=sf.ops.zero())
        g.wait_all()
        for d in range(ndev):
            torch.cuda.synchronize(d)
        if rep == args.warmup:
            clocks.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        parts = alg.insert_particles(g, P, F, partials=parts)
        g.wait_all()
        e1.record()
        torch.cuda.synchronize()
        if rep >= args.warmup:
            times.append(e0.elapsed_time(e1) / 1e3)
    clk = clocks.stop()
    stats = [eng.stats(d) for d in range(ndev)]
    eng.stop()
    t = statistics.mean(times)
    inter = alg.interactions(ng * per)
    bound = ndev * dfma_tf * 1e12 / 2 / 11.5
    line = {
        "metric": "particle interactions/s (C4, FP64)", "value": inter / t, "unit": "interactions/s",
        "n_gpus": ndev, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (positions uniform in the unit cube, charges in [0.5, 1], generated on device)",
        "config": {"workload": f"particles {ng * per} in {ng} groups, 32896 tasks, {ndev} GPU(s) from one runtime",
                   "parallelism": "pair tasks in balanced blocks per GPU, per-GPU partial accumulators, "
                                  "dacc reduction (peer pulls)", "l2": "one evaluation per step"},
        "clocks": clk,
        "roofline": {"bound": "fp64 pipe", "achieved": inter / t, "peak": bound, "unit": "interactions/s",
                     "frac": inter / t / bound, "dfma_peak_tflops_per_gpu": dfma_tf},
        "p2p_bytes": sum(s["bytes_p2p_in"] for s in stats),
        "gpu_launches": stats[0]["kernel_launches"],
    }
    print(json.dumps(line), flush=True)
    dist.barrier()


def main():
    args = parse()
    dist = Dist()
    if args.impl == "reference":
        run_reference(args, dist)
        return
    dist.init("nccl")
    if args.workload == "cholesky":
        main_cholesky(args, dist)
    elif args.workload == "particles":
        main_particles(args, dist)
    else:
        args.n, args.b = args.n or 16384, args.b or 512
        main_ours(args, dist)
    dist.done()


if __name__ == "__main__":
    main()
