#!/usr/bin/env python
"""Benchmark of the STF GPU execution path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one process per GPU)

Workload by GPU count (``--workload auto``, the default):

  N = 1   BASELINE.json configs[1] (C2): tiled DGEMM 16384 x 16384 FP64 with
          512 x 512 tiles ("1024 tiles") -> 32,768 GEMM tasks per step, inserted
          through the drop-in TaskGraph API and executed by the native runtime.
          Inputs (3 x 2 GiB) are far larger than the 126 MB L2: no flush needed.
  N > 1   BASELINE.json configs[2] (C3): tiled Cholesky 32768 x 32768 / 1024
          tiles over all N GPUs from ONE runtime (rank 0): 2-D block-cyclic
          owner-computes placement, panels pulled peer-to-peer over NVLink
          (strong scaling).  The same run also factors C3 on GPU 0 alone so
          the line carries its own 1-GPU reference; at N >= 8 it adds the
          north-star C5 leg (65536 / 1024 tiles on all N GPUs and on one).
          Fewer visible GPUs than N is an error (no silent fallback to one GPU).

Legs of the N = 1 JSON line:
  value         device-resident inputs, FP64 GFLOP/s (CUDA events, max over ranks)
  check         every leg verifies its output after its timed region (verify.py):
                sampled C tiles vs numpy, the C3 randomized residual, sampled
                C4 particles; the tolerances and the errors are in the line
  e2e           same metric through the public API from pinned HOST buffers: every
                step stages A, B, C host->device on demand and flushes C back;
                achieved H2D / D2H GB/s next to the measured PCIe rates
  roofline      FP64 DMMA pipe: achieved TFLOP/s of the DGEMM kernel over the
                timed region vs the DMMA peak measured in-run on this GPU
  cpu_baseline  the reference algorithm on the host cores (oracle restatement of
                the reference STF engine + numpy bodies; rank 0, N=1), bounded
                samples of C2 (headline), C1, C3 and C4, and the reference's
                overhead protocol on the same cores
  secondary     C1, C3 (with residual) and C4 (with sampled check) on one GPU,
                and the runtime overhead in us/task: the reference protocol
                (src/bench.py:67-117) with T = host cores, N = 1000,
                D in {0, 1e-4, 1e-3} s, write and commute, deps in {1, 5, 20}
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

import verify  # noqa: E402  (numpy output checkers; no oracle)

METRIC = "FP64 GFLOP/s tiled Cholesky/GEMM at 1/2/4/8 B200 (% FP64 peak); µs/task"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=("auto", "gemm", "cholesky", "particles"), default="auto",
                    help="auto: gemm (C2) at N=1, cholesky (C3) over N GPUs at N>1; cholesky/particles run "
                         "over all --gpus GPUs from one runtime")
    ap.add_argument("--ordinals", default=None,
                    help="comma-separated CUDA ordinals for the multi-GPU legs (e.g. 0,0 = two logical "
                         "devices on one GPU, for functional runs on a 1-GPU box)")
    ap.add_argument("--n", "--matrix-n", dest="n", type=int, default=None)
    ap.add_argument("--b", "--tile-b", dest="b", type=int, default=None)
    ap.add_argument("--streams", type=int, default=32)
    ap.add_argument("--group", type=int, default=32)
    ap.add_argument("--chol-group", type=int, default=8,
                    help="launch-group size for the Cholesky legs (tools/chol_sweep.py: 8 best for b=1024)")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--e2e-skew", type=int, default=-1, help="insert_gemm skew on the e2e leg (-1: 3 nt, 0: FIFO)")
    ap.add_argument("--pipeline", type=int, default=1,
                    help="device-resident leg: the K steps inserted back to back in one timed bracket (0: per step)")
    ap.add_argument("--e2e-pipeline", type=int, default=1,
                    help="e2e headline: steps inserted back to back with one wait at the end (0: per-step wait)")
    ap.add_argument("--e2e-stage-stream", type=int, default=1,
                    help="e2e leg: host staging copies on the copy stream (runtime option stage_stream)")
    ap.add_argument("--e2e-stage-window", type=int, default=0,
                    help="e2e leg: runtime option stage_window in MiB (0: off)")
    ap.add_argument("--e2e-flush-priority", type=int, default=0, help="e2e leg: runtime option flush_priority")
    ap.add_argument("--e2e-skew-block", type=int, default=-1,
                    help="insert_gemm skew_block on the e2e leg (-1: nt / 2, 0: row-major chain offsets)")
    ap.add_argument("--e2e-tile-block", type=int, default=0, help="insert_gemm tile_block on the e2e leg (overrides skew)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--overhead-n", type=int, default=1000)
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
            import datetime

            # ranks > 0 of the multi-GPU Cholesky line wait in a barrier while rank 0
            # drives every GPU (C3, its 1-GPU reference and at N >= 8 the C5 leg)
            dist.init_process_group(backend, timeout=datetime.timedelta(minutes=30))
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

    def __init__(self, index):
        self.index = index if isinstance(index, (list, tuple)) else [index]
        self.samples = []
        self._stop = threading.Event()
        self._th = None
        self._proc = None

    def start(self):
        # ONE long-running `nvidia-smi ... -lms 200` (the profiling recipe's clocks
        # line), not a process per sample: spawning nvidia-smi every 0.2 s costs a
        # driver/NVML initialisation each time on the host the runtime runs on
        ids = ",".join(str(i) for i in sorted(set(self.index)))
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", ids, "--query-gpu=" + self.FIELDS,
                                           "--format=csv,noheader,nounits", "-lms", "200"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self._proc = None
            return self

        def run():
            try:
                for line in self._proc.stdout:
                    if self._stop.is_set():
                        break
                    line = line.strip()
                    if line:
                        self.samples.append([x.strip() for x in line.split(",")])
            except Exception:
                pass

        self._th = threading.Thread(target=run, daemon=True)
        self._th.start()
        return self

    def stop(self):
        self._stop.set()
        proc = getattr(self, "_proc", None)
        if proc is not None:
            proc.terminate()
            try:
                proc.wait(timeout=10)
            except Exception:
                proc.kill()
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


# ------------------------------------------------- overhead protocol (both arms)

def derive_report(t0: int, insertion_ns: int, ends, duration: float) -> dict:
    """Per-rep numbers from raw end timestamps, restated from the reference's
    src/bench.py:96-117 (O_avg = makespan / N - D; O_max = worst gap between
    consecutive ends of a chain minus D; insertion cost per task)."""
    T = len(ends)
    N = len(ends[0])
    makespan_s = (max(max(row) for row in ends) - t0) / 1e9
    o_max = None
    for row in ends:
        prev = t0
        for end in sorted(row):
            gap = (end - prev) / 1e9 - duration
            o_max = gap if o_max is None or gap > o_max else o_max
            prev = end
    return {"insertion_per_task_us": insertion_ns / 1e3 / (T * N), "makespan_s": makespan_s,
            "o_avg_us": (makespan_s / N - duration) * 1e6, "o_max_us": o_max * 1e6}


def _mean_reports(reps):
    return {k: statistics.mean(r[k] for r in reps) for k in reps[0]}


def overhead_gpu(sf, dev, T, N, D, mode, deps, reps=3):
    """The reference overhead protocol on the GPU engine: T chains (CUDA streams)
    x N tasks, each writing (or commutatively writing) its chain cell and reading
    deps-1 extra cells; the body is a D-second device spin (no kernel at D = 0).
    End timestamps are the tasks' CUDA end events on the host clock."""
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, T), trace=True, ordinals=[dev], device_memory=1 << 26)
    acc = sf.write if mode == "write" else sf.commutative_write
    op = sf.ops.noop if D == 0 else sf.ops.spin(int(D * 1e9))
    out = []
    try:
        for _ in range(reps + 1):  # the first rep warms the streams / event pools
            g = sf.TaskGraph().compute_on(eng)
            chains = [sf.Cell(0) for _ in range(T)]
            extras = [[sf.Cell(0) for _ in range(deps - 1)] for _ in range(T)]
            for c in range(T):  # stage the cells before the clock starts (the reference's are host objects)
                g.task(sf.write(chains[c]), *[sf.write(x) for x in extras[c]], device=sf.ops.noop)
            g.wait_all()
            owner = {}
            t0 = time.perf_counter_ns()
            for i in range(N):
                for c in range(T):
                    v = g.task(acc(chains[c]), *[sf.read(x) for x in extras[c]], device=op)
                    owner[v.task_id] = (c, i)
            ins = time.perf_counter_ns() - t0
            g.wait_all()
            ends = [[0] * N for _ in range(T)]
            for kind, t, _, tid, _ in g.trace.export_events():
                if kind == "TaskEnd" and tid in owner:
                    c, i = owner[tid]
                    ends[c][i] = t + g._t0  # export_events is relative to the graph's t0
            out.append(derive_report(t0, ins, ends, D))
    finally:
        eng.stop()
    return _mean_reports(out[1:])


def overhead_cpu(T, N, D, mode, deps, reps=2):
    """The same protocol on the oracle restatement of the reference engine (host
    worker threads, precise-sleep bodies as in the reference)."""
    from oracle import stf

    m = stf.WRITE if mode == "write" else stf.COMMUTE
    out = []

    def precise_sleep(d):  # reference src/bench.py:29-37
        if d <= 0:
            return
        deadline = time.perf_counter() + d
        if d > 200e-6:
            time.sleep(d - 150e-6)
        while time.perf_counter() < deadline:
            time.sleep(0)

    for _ in range(reps):
        orc = stf.Oracle(workers=T, trace=False)
        chains = [[0] for _ in range(T)]
        extras = [[[0] for _ in range(deps - 1)] for _ in range(T)]
        ends = [[0] * N for _ in range(T)]

        def body(c, i):
            row = ends[c]

            def run(*_):
                precise_sleep(D)
                row[i] = time.perf_counter_ns()
            return run

        t0 = time.perf_counter_ns()
        for i in range(N):
            for c in range(T):
                orc.task([(m, chains[c])] + [(stf.READ, x) for x in extras[c]], body=body(c, i))
        ins = time.perf_counter_ns() - t0
        orc.wait_all()
        orc.stop()
        out.append(derive_report(t0, ins, ends, D))
    return _mean_reports(out)


OVERHEAD_GRID = [(D, mode, 1) for D in (0.0, 1e-4, 1e-3) for mode in ("write", "commute")] + \
                [(1e-4, mode, deps) for deps in (5, 20) for mode in ("write", "commute")]


def overhead_rows(fn, T, N):
    rows = []
    for D, mode, deps in OVERHEAD_GRID:
        r = fn(T, N, D, mode, deps)
        r.update({"D_s": D, "mode": mode, "deps": deps, "T": T, "N": N})
        rows.append(r)
    return rows


# ----------------------------------------------------------------- CPU legs

def cpu_baseline(n: int, b: int, seconds: float, steps: int = 1, warmup: int = 0, extra: bool = True,
                 overhead_n: int = 1000):
    """Reference algorithm on the host: the oracle's restatement of the reference
    STF engine (one worker thread per core) running numpy tile bodies, on the
    first block-rows of the same tiled DGEMM (bounded sample).  One calibration
    pass sizes the sample to about `seconds`; then `warmup` untimed and `steps`
    timed samples run, and the mean rate of the timed ones is returned.  With
    ``extra``: C1 in full and bounded samples of C3 / C4, plus the reference
    overhead protocol on the same cores."""
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
    out = {"value": flops / dt / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "port",
           "library_ceiling_gflops": lib, "library_ceiling": f"numpy/OpenBLAS {m}^2 FP64 A@B, all host threads",
           "sample": f"tiled DGEMM {n}/{b}: block-rows 0..{rows - 1} of C ({rows * nt * nt} tasks, "
                     f"{flops / 1e12:.2f} TFLOP per sample) on the oracle STF engine (restated reference, "
                     f"{cores} host worker threads, numpy bodies, 1 BLAS thread each); "
                     f"{len(dts)} timed sample(s), mean",
           "seconds": dt}
    if extra:
        with threadpool_limits(1):
            out["configs"] = cpu_configs(cores)
        out["overhead"] = {"protocol": "reference src/bench.py:67-117 on the oracle engine, host worker threads, "
                                       "precise-sleep bodies", "runs": overhead_rows(overhead_cpu, cores, overhead_n)}
    return out


def cpu_configs(cores):
    """C1 in full, and the first panel steps of C3 / the first pair tasks of C4,
    on the oracle engine with numpy bodies (1 BLAS thread per worker)."""
    import numpy as np

    from oracle import inputs, programs, stf

    res = {}
    # C1: DGEMM 2048 / 256, all 512 tasks
    n, b = 2048, 256
    objs = programs.gemm_operands(n, b)
    t0 = time.perf_counter()
    programs.run_on_oracle(programs.gemm_program(n // b), objs, workers=cores, trace=False).stop()
    dt = time.perf_counter() - t0
    res["C1"] = {"gflops": 2.0 * n ** 3 / dt / 1e9, "seconds": dt, "sample": "full (512 tasks)"}
    # C3: Cholesky 32768 / 1024, panel steps 0..2 (the first 1,488 tasks)
    n, b, steps = 32768, 1024, 3
    nt = n // b
    prog = [t for t in programs.cholesky_program(nt)]
    cut = []
    for kind, acc, prio in prog:
        if kind == "potrf" and acc[0][1][1] >= steps:
            break
        cut.append((kind, acc, prio))
    keys = {key for _, acc, _ in cut for _, key in acc}
    objs = {key: inputs.spd_tile(3, key[1] * b, key[2] * b, b, b, n) for key in keys}
    t0 = time.perf_counter()
    programs.run_on_oracle(cut, objs, workers=cores, trace=False).stop()
    dt = time.perf_counter() - t0
    fl = programs.flops(cut, b)
    res["C3"] = {"gflops": fl / dt / 1e9, "seconds": dt,
                 "sample": f"panel steps 0..{steps - 1} of C3 ({len(cut)} of 5984 tasks, {fl / 1e12:.2f} TFLOP)"}
    # C4: particles 2^20 / 256 groups: the first 3 * cores pair tasks
    per = 4096
    npairs = 3 * cores
    P = [inputs.particles(4, g * per, per) for g in range(npairs + 1)]
    F = [np.zeros((4, per)) for _ in range(npairs + 1)]
    orc = stf.Oracle(workers=cores, trace=False)
    from oracle import bodies
    t0 = time.perf_counter()
    for j in range(1, npairs + 1):
        orc.task([(stf.READ, P[0]), (stf.READ, P[j]), (stf.COMMUTE, F[0]), (stf.COMMUTE, F[j])],
                 body=bodies.p2p_pair)
    orc.wait_all()
    dt = time.perf_counter() - t0
    orc.stop()
    inter = 2.0 * per * per * npairs
    res["C4"] = {"interactions_per_s": inter / dt, "seconds": dt,
                 "sample": f"{npairs} pair tasks of 4096 x 4096 particles (mutual)"}
    return res


def run_reference(args, dist):
    """The reference arm: the reference algorithm on the host cores (the oracle
    port of the reference STF engine + numpy bodies), same metric and config as
    our arm at this N.  Under torchrun only rank 0 runs."""
    if dist.rank != 0:
        return
    workload = resolve_workload(args, max(args.gpus, dist.world))
    per_step = max(1.0, min(args.cpu_seconds, 150.0 / max(1, args.steps + args.warmup)))
    if workload == "gemm":
        args.n, args.b = args.n or 16384, args.b or 512
        res = cpu_baseline(args.n, args.b, per_step, steps=args.steps, warmup=args.warmup, extra=False)
        nt = args.n // args.b
        cfg = {"workload": f"tiled DGEMM {args.n}x{args.n} fp64, {args.b}x{args.b} tiles (BASELINE configs[1], "
                           f"C2), {nt ** 3} GEMM tasks per step per GPU", "n": args.n, "b": args.b,
               "cpu_sample": res["sample"]}
        value, seconds, sample = res["value"], res["seconds"], res["sample"]
    else:
        from threadpoolctl import threadpool_limits

        with threadpool_limits(1):
            c3 = cpu_configs(os.cpu_count() or 1)["C3"]
        value, seconds, sample = c3["gflops"], c3["seconds"], c3["sample"]
        cfg = {"workload": "tiled Cholesky 32768x32768 fp64, 1024x1024 tiles (BASELINE configs[2], C3)",
               "n": 32768, "b": 1024, "cpu_sample": sample}
    cores = os.cpu_count() or 1
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": seconds * 1e3,
        "higher_is_better": True, "scaling": "weak" if workload == "gemm" else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU legs

def pcie_rates(dev: int):
    """Pinned host <-> device copy rates (GB/s) with CUDA events, 1 GiB each way."""
    import torch

    nbytes = 1 << 30
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{dev}")
    out = {}
    for name, (dst, src) in (("h2d", (d, h)), ("d2h", (h, d))):
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize(dev)
        out[name] = 3 * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9
    del h, d
    return out


def gemm_check(g, A, B, C, mult, seed):
    """Flush A, B, C (read mode: device copies stay) and check sampled C tiles."""
    for M in (A, B, C):
        for t in M.tiles.values():
            g.flush_to_host(t, keep_device=True)
    g.wait_all()
    samples = verify.sample_tiles(A.nt, 4, seed=seed)
    rel, comp = verify.gemm_tile_errors(C.tiles, A.tiles, B.tiles, samples, mult=mult)
    tol_c = verify.gemm_componentwise_tol(A.nt * A.b, mult)
    return {"tiles_checked": len(samples), "max_rel_err": rel, "max_componentwise_err": comp,
            "tol_rel": verify.GEMM_REL_TOL, "tol_componentwise": tol_c,
            "expected": f"C = {mult:g} * A B", "pass": rel <= verify.GEMM_REL_TOL and comp <= tol_c}


def main_gemm(args, dist):
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

    for _ in range(args.warmup):
        step()
    iso = []
    if args.pipeline:  # the same step timed alone (insert, wait) after the warm-up, for comparison
        for _ in range(2):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step()
            e1.record()
            torch.cuda.synchronize()
            iso.append(e0.elapsed_time(e1) / 1e3)
    st0 = eng.stats(0)
    p0 = sf.gemm_paths()
    clocks = ClockSampler(dev).start()
    times = []
    if args.pipeline:
        # the K steps in ONE bracket, inserted back to back with one wait at the end:
        # step k+1's chain on a C tile starts when step k's chain on it ends, so the
        # steps' ramp-down and ramp-up overlap (ms_per_step = total / K)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            alg.insert_gemm(g, A, B, C)
        g.wait_all()
        e1.record()
        torch.cuda.synchronize()
        times = [e0.elapsed_time(e1) / 1e3 / args.steps] * args.steps
    else:
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
    p1 = sf.gemm_paths()
    step_s = dist.max(statistics.mean(times))
    value = flops * dist.world / step_s / 1e9
    launches = st1["kernel_launches"] - st0["kernel_launches"]
    check = None if args.no_check else gemm_check(g, A, B, C, float(args.warmup + args.steps + len(iso)), seed=1)

    # ---- e2e: host-resident inputs through the public API ----
    def e2e_step(wait=True, prio_base=0):
        # wavefront priorities (insert_gemm skew): the k-chains of the C tiles start
        # staggered, so C's staging (2 GiB H2D) and its flush (2 GiB D2H) spread
        # over the step instead of piling up in the first and last waves (round 1,
        # tools/e2e_probe.py: 25.7 -> 28.3 TFLOP/s).  Round 2 (tools/e2e_timeline.py,
        # profiles/r2_e2e_timeline.md): the chains take their offsets in nt/2 x nt/2
        # blocks (the first waves share half the rows of A and columns of B: more
        # tasks per staged tile while PCIe is the bottleneck), spread over 3 nt
        # waves, and the staging copies run in one FIFO on the copy stream
        # (stage_stream): 29.8-30.2 -> 30.8-31.2 TFLOP/s.
        if args.e2e_tile_block:
            alg.insert_gemm(g, A, B, C, tile_block=args.e2e_tile_block)
        else:
            alg.insert_gemm(g, A, B, C, skew=args.e2e_skew if args.e2e_skew >= 0 else 3 * nt,
                            skew_block=args.e2e_skew_block if args.e2e_skew_block >= 0 else max(1, nt // 2),
                            prio_base=prio_base)
        for t in C.tiles.values():
            g.flush_to_host(t)                      # C back to the host (write-mode flush)
        for M in (A, B):
            for t in M.tiles.values():
                g.flush_to_host(t)                  # clean copies dropped: next step restages
        if wait:
            g.wait_all()

    # more launch groups queued per stream keeps the copy engines and the SMs both
    # busy while tiles stream in (tools/e2e_probe.py: 22.4 -> 25.5-26 TFLOP/s)
    eng.set_option("groups_per_stream", 4)
    # the launch-group timing events serve the kernel roofline only (device leg);
    # the e2e leg runs the product configuration without them
    eng.set_option("kernel_timing", 0)
    eng.set_option("stage_stream", args.e2e_stage_stream)
    eng.set_option("stage_window", args.e2e_stage_window << 20)
    eng.set_option("flush_priority", args.e2e_flush_priority)
    e2e_step()  # first pass moves everything to the host side
    s0 = eng.stats(0)
    et = []
    ke = max(2, args.steps // 2)
    for _ in range(ke):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        e2e_step()
        e1.record()
        torch.cuda.synchronize()
        et.append(e0.elapsed_time(e1) / 1e3)
    s1 = eng.stats(0)
    iso_s = dist.max(statistics.mean(et))
    h2d = (s1["bytes_to_device"] - s0["bytes_to_device"]) // ke
    d2h = (s1["bytes_from_device"] - s0["bytes_from_device"]) // ke
    kp = 0
    e2e_s = iso_s
    if args.e2e_pipeline:
        # the same steps inserted back to back with ONE wait at the end (a user
        # streaming batches): step k+1's tasks on a tile wait only for step k's
        # flush of THAT tile, so its staging overlaps step k's last chains instead
        # of every step paying its own cold start and tail.  Every step still
        # stages its A, B, C host->device and flushes C device->host.
        kp = max(3, args.steps)
        s2 = eng.stats(0)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for q in range(kp):
            # each product strictly below the previous one in priority
            e2e_step(wait=False, prio_base=-q * (4 * nt + 1))
        g.wait_all()
        e1.record()
        torch.cuda.synchronize()
        e2e_s = dist.max(e0.elapsed_time(e1) / 1e3 / kp)
        s3 = eng.stats(0)
        h2d = (s3["bytes_to_device"] - s2["bytes_to_device"]) // kp
        d2h = (s3["bytes_from_device"] - s2["bytes_from_device"]) // kp
    e2e = {"value": flops * dist.world / e2e_s / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3,
           "timing": (f"{kp} steps inserted back to back, one wait_all at the end (ms_per_step = total / {kp})"
                      if kp else f"{ke} steps, each followed by wait_all (mean)"),
           "isolated_step": {"value": flops * dist.world / iso_s / 1e9, "ms_per_step": iso_s * 1e3,
                             "steps": ke, "how": "each step timed alone: insert, flush, wait_all"},
           "h2d_gbs": h2d / e2e_s / 1e9, "d2h_gbs": d2h / e2e_s / 1e9,
           "schedule": ({"tile_block": args.e2e_tile_block} if args.e2e_tile_block else
                        {"skew": args.e2e_skew if args.e2e_skew >= 0 else 3 * nt,
                         "skew_block": args.e2e_skew_block if args.e2e_skew_block >= 0 else max(1, nt // 2)})
           | {"stage_stream": args.e2e_stage_stream, "stage_window_mib": args.e2e_stage_window,
              "flush_priority": args.e2e_flush_priority, "groups_per_stream": 4}}
    if not args.no_check:
        # the host now holds C = (warmup + steps + 1 + ke) A B (every e2e pass accumulates)
        samples = verify.sample_tiles(nt, 3, seed=2)
        rel, comp = verify.gemm_tile_errors(C.tiles, A.tiles, B.tiles, samples,
                                            mult=float(args.warmup + args.steps + len(iso) + 1 + ke + kp))
        tol_c = verify.gemm_componentwise_tol(n, args.warmup + args.steps + len(iso) + 1 + ke + kp)
        e2e["check"] = {"tiles_checked": len(samples), "max_rel_err": rel, "max_componentwise_err": comp,
                        "tol_rel": verify.GEMM_REL_TOL, "tol_componentwise": tol_c,
                        "pass": rel <= verify.GEMM_REL_TOL and comp <= tol_c}
    eng.stop()
    del A, B, C
    try:
        pc = pcie_rates(dev)
        e2e["pcie_h2d_gbs"], e2e["pcie_d2h_gbs"] = pc["h2d"], pc["d2h"]
        e2e["transfer_note"] = ("h2d_gbs / d2h_gbs: bytes moved per e2e step / step time (copies overlap the "
                                "kernels); pcie_*_gbs: 1 GiB pinned copies alone, CUDA events")
    except Exception as exc:  # the probe must not hide the line
        e2e["pcie_error"] = repr(exc)

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
    paths = {k: p1[k] - p0[k] for k in p1}
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
                "kernel_paths": paths,
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
        "clocks": clk, "check": check, "e2e": e2e, "gpu_launches": launches, "roofline": roofline,
        "pct_fp64_peak": 100.0 * value / dist.world / 1e3 / peak_tf,
        "runtime_host_us_per_task": {k: (st1[k] - st0[k]) / 1e3 / max(1, st1["tasks_executed"] - st0["tasks_executed"])
                                     for k in ("t_plan_ns", "t_issue_ns", "t_release_ns", "t_complete_ns")}
        | {"stream_waits_per_task": (st1["stream_waits"] - st0["stream_waits"]) /
           max(1, st1["tasks_executed"] - st0["tasks_executed"]), "host_cores": os.cpu_count()},
        "timing": (f"{args.steps} steps inserted back to back in one bracket, one wait_all (ms_per_step = total / "
                   f"{args.steps})" if args.pipeline else f"{args.steps} steps, each bracketed and waited"),
        "isolated_step": ({"value": flops * dist.world / dist.max(statistics.mean(iso)) / 1e9,
                           "ms_per_step": 1e3 * dist.max(statistics.mean(iso)), "steps": len(iso)} if iso else None),
    }

    if dist.rank == 0 and dist.world == 1 and not args.no_secondary:
        line["secondary"] = secondary(sf, alg, dev, args, peak_tf)
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu:
        try:
            cb = cpu_baseline(n, b, args.cpu_seconds, overhead_n=args.overhead_n)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                       "library_ceiling_gflops", "library_ceiling", "configs",
                                                       "overhead")}
        except Exception as exc:  # the CPU leg must not hide the GPU line
            line["cpu_baseline"] = {"error": repr(exc)}
    if dist.rank == 0:
        print(json.dumps(line), flush=True)


def cholesky_run(sf, alg, ordinals, n, b, streams, group, reps, check, clocks=None, timed_from=None,
                 e2e_reps=0):
    """Factor C3-style SPD matrices ``reps`` times on the given devices from one
    runtime (block-cyclic when several); returns per-rep seconds, the runtime
    counters summed over reps ``timed_from`` .. reps-1 (default: the last rep) and
    the residual of the last rep.  ``e2e_reps`` > 0 adds an end-to-end leg
    (returned as a 4th value): the SPD input starts on the HOST (flushed there,
    device copies dropped), each timed rep stages it on demand, factors and
    flushes L back to the host."""
    if timed_from is None:
        timed_from = reps - 1
    import torch

    ndev = len(ordinals)
    mem = None
    if len(set(ordinals)) < ndev:
        # logical devices sharing a GPU (host-side scaling runs): split its free HBM
        # (the per-device streams' scratch and the cooperative kernels' workspaces
        # come out of the headroom left beside the arenas: 2 GiB per logical device)
        mem = [int((torch.cuda.mem_get_info(o)[0] - (6 << 30) - ordinals.count(o) * (2 << 30)) /
                   ordinals.count(o)) for o in ordinals]
    eng = sf.create_engine(sf.WorkerTeam.of_devices(ndev, streams), scheduler="prio", trace=False,
                           ordinals=list(ordinals), group_max=group, device_memory=mem)
    M = alg.TiledMatrix(n, b, lower=True)
    P, Q = alg.grid_shape(ndev)
    times = []
    A = None
    res = None
    try:
        s_before = None
        g = sf.TaskGraph().compute_on(eng)  # one graph: the tiles keep their handles across reps
        if ndev > 1:
            alg.block_cyclic(g, M, P, Q)
        for rep in range(reps):
            alg.insert_fill_spd(g, M, 3)
            if check and rep == reps - 1:
                g.flush_all(keep_device=True)
            g.wait_all()
            if check and rep == reps - 1:
                A = {ij: t.copy() for ij, t in M.tiles.items()}
            for o in set(ordinals):
                torch.cuda.synchronize(o)
            if rep == 1 and clocks is not None:
                clocks.start()
            if rep == timed_from:
                s_before = [eng.stats(d) for d in range(ndev)]
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            alg.insert_cholesky(g, M)
            g.wait_all()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        stats = [eng.stats(d) for d in range(ndev)]
        delta = [{k: s1[k] - s0[k] for k in ("bytes_p2p_in", "copies_p2p_in", "tasks_executed", "t_plan_ns",
                                             "t_issue_ns", "t_complete_ns", "groups", "kernel_launches")}
                 for s0, s1 in zip(s_before, stats)]
        if check:
            g.flush_all(keep_device=False)
            g.wait_all()
            res = verify.cholesky_residual(A, M.tiles, n, b)
        e2e = None
        if e2e_reps:
            et = []
            h2d = d2h = 0
            for r in range(e2e_reps + 1):  # the first rep is a warm-up
                alg.insert_fill_spd(g, M, 3)
                g.flush_all(keep_device=False)  # the input now lives on the host only
                g.wait_all()
                for o in set(ordinals):
                    torch.cuda.synchronize(o)
                e_before = [eng.stats(d) for d in range(ndev)]
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                alg.insert_cholesky(g, M)       # stages every tile host -> device on demand
                g.flush_all(keep_device=False)  # L back to the host
                g.wait_all()
                e1.record()
                torch.cuda.synchronize()
                e_after = [eng.stats(d) for d in range(ndev)]
                if r >= 1:  # bytes of the timed region only (the fill and input flush are outside)
                    et.append(e0.elapsed_time(e1) / 1e3)
                    h2d += sum(a["bytes_to_device"] - z["bytes_to_device"] for z, a in zip(e_before, e_after))
                    d2h += sum(a["bytes_from_device"] - z["bytes_from_device"] for z, a in zip(e_before, e_after))
            e2e = {"seconds": statistics.mean(et), "h2d_bytes_per_step": h2d // e2e_reps,
                   "d2h_bytes_per_step": d2h // e2e_reps}
    finally:
        eng.stop()
    if e2e_reps:
        return times, delta, res, e2e
    return times, delta, res


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
    ordinals = [int(x) for x in args.ordinals.split(",")] if args.ordinals else list(range(ndev))
    if len(ordinals) != ndev:
        raise SystemExit(f"--ordinals names {len(ordinals)} devices but --gpus is {ndev}")
    visible = torch.cuda.device_count()
    if max(ordinals) >= visible:
        raise SystemExit(f"bench: {ndev} GPUs requested but only {visible} visible (no fallback to fewer GPUs)")
    n, b = args.n or 32768, args.b or 1024
    nt = n // b
    peak_tf, _ = sf.fp64_peak(ordinals[0])
    flops = alg.flops_cholesky(n)
    clocks = ClockSampler(ordinals)
    times, delta, res, ce2e = cholesky_run(sf, alg, ordinals, n, b, args.streams, args.chol_group,
                                           args.warmup + args.steps, not args.no_check, clocks,
                                           timed_from=args.warmup, e2e_reps=2)
    clk = clocks.stop()
    t = statistics.mean(times[args.warmup:])
    value = flops / t / 1e9
    one = None
    if ndev > 1:
        # the 1-GPU reference of the scaling curve, measured in the same run
        t1, _, _ = cholesky_run(sf, alg, [ordinals[0]], n, b, args.streams, args.chol_group, 4, False)
        one = {"n_gpus": 1, "value": flops / statistics.mean(t1[2:]) / 1e9, "unit": "GFLOP/s",
               "ms_per_step": 1e3 * statistics.mean(t1[2:])}
    north = None
    if ndev >= 8 and not args.no_secondary:
        # the north-star configuration (BASELINE configs[4], C5): N = 65536 / 1024
        # tiles over the same devices, with its own 1-GPU reference and residual
        n5 = 65536
        f5 = alg.flops_cholesky(n5)
        t5, d5, r5 = cholesky_run(sf, alg, ordinals, n5, b, args.streams, args.chol_group, 3, not args.no_check)
        t51, _, _ = cholesky_run(sf, alg, [ordinals[0]], n5, b, args.streams, args.chol_group, 2, False)
        v5 = f5 / statistics.mean(t5[1:]) / 1e9
        v51 = f5 / t51[-1] / 1e9
        north = {"workload": f"tiled Cholesky {n5}x{n5} fp64, {b}x{b} tiles (BASELINE configs[4], C5), "
                             f"{ndev} GPU(s) from one runtime",
                 "value": v5, "unit": "GFLOP/s", "ms_per_step": 1e3 * statistics.mean(t5[1:]),
                 "frac_aggregate_fp64_peak": v5 / 1e3 / (peak_tf * ndev),
                 "one_gpu_value": v51, "speedup_vs_one_gpu": v5 / v51,
                 "target": ">= 0.60 of aggregate FP64 peak and >= 6x over 1 GPU (BASELINE north_star)",
                 "p2p_bytes_per_step": sum(d["bytes_p2p_in"] for d in d5),
                 "rep_ms": [round(1e3 * x, 2) for x in t5],
                 "check": None if r5 is None else {"cholesky_residual": r5, "tol": verify.CHOL_RESIDUAL_TOL,
                                                   "pass": r5 <= verify.CHOL_RESIDUAL_TOL}}
    ntasks = nt + nt * (nt - 1) + nt * (nt - 1) * (nt - 2) // 6  # potrf + trsm + syrk + gemm
    p2p = sum(d["bytes_p2p_in"] for d in delta) / args.steps  # delta covers the timed reps
    tasks = sum(d["tasks_executed"] for d in delta)
    launches = sum(d["kernel_launches"] for d in delta)
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ndev, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic SPD (R+R^T)/2 + n*I, generated on device",
        "config": {"workload": f"tiled Cholesky {n}x{n} fp64, {b}x{b} tiles (BASELINE configs[2], C3), "
                               f"{ntasks} tasks, {ndev} GPU(s) from one runtime",
                   "n": n, "b": b, "tasks": ntasks, "grid": list(alg.grid_shape(ndev)),
                   "ordinals": ordinals, "streams_per_gpu": args.streams,
                   "parallelism": "owner-computes 2-D block-cyclic, NVLink peer pulls",
                   "l2": "working set (%.1f GiB) larger than L2" % (nt * (nt + 1) / 2 * b * b * 8 / 2 ** 30)},
        "clocks": clk,
        "check": None if res is None else {"cholesky_residual": res, "tol": verify.CHOL_RESIDUAL_TOL,
                                           "pass": res <= verify.CHOL_RESIDUAL_TOL,
                                           "how": "||A x - L L^T x|| / (||A||_F ||x||), 4 seeded x"},
        "pct_fp64_peak": 100.0 * value / 1e3 / (peak_tf * ndev),
        "roofline": {"bound": "tensor", "achieved": value / 1e3 / ndev, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": value / 1e3 / ndev / peak_tf, "traffic": None,
                     "peak_source": "FP64 DMMA peak measured in-run (sfx_fp64_peak), per GPU"},
        "scaling_reference": one,
        "north_star_C5": north,
        "e2e": {"value": flops / ce2e["seconds"] / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": ce2e["h2d_bytes_per_step"], "d2h_bytes_per_step": ce2e["d2h_bytes_per_step"],
                "ms_per_step": 1e3 * ce2e["seconds"],
                "how": "SPD input on the host (pinned tiles, device copies dropped); each step stages it on "
                       "demand, factors on all GPUs and flushes L back (flush_all), 2 steps after 1 warm-up"},
        "p2p": {"bytes_per_step": p2p, "gbs": p2p / t / 1e9,
                "per_gpu_bytes": [d["bytes_p2p_in"] // args.steps for d in delta]},
        "runtime_host_us_per_task": {k: sum(d[k] for d in delta) / 1e3 / max(tasks, 1)
                                     for k in ("t_plan_ns", "t_issue_ns", "t_complete_ns")},
        "rep_ms": [round(1e3 * x, 2) for x in times],
        "gpu_launches": launches,  # this process's kernels over the timed factorizations, all GPUs
    }
    print(json.dumps(line), flush=True)
    dist.barrier()


def secondary(sf, alg, dev, args, peak_tf):
    import torch

    out = {}
    # C1: DGEMM 2048 / 256 (the oracle-run config) on the GPU, checked
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 16), scheduler="prio", trace=False, ordinals=[dev])
    n, b = 2048, 256
    A, B, C = (alg.TiledMatrix(n, b) for _ in range(3))
    g = sf.TaskGraph().compute_on(eng)
    alg.insert_fill_uniform(g, A, 1)
    alg.insert_fill_uniform(g, B, 2)
    alg.insert_zero(g, C)
    g.wait_all()
    ts = []
    for rep in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        alg.insert_gemm(g, A, B, C)
        g.wait_all()
        e1.record()
        torch.cuda.synchronize()
        if rep:
            ts.append(e0.elapsed_time(e1) / 1e3)
    t = statistics.mean(ts)
    out["dgemm_C1"] = {"n": n, "b": b, "tasks": 512, "seconds": t, "gflops": alg.flops_gemm(n) / t / 1e9,
                       "check": gemm_check(g, A, B, C, 4.0, seed=4)}
    eng.stop()
    del A, B, C
    # C3: tiled Cholesky 32768 / 1024 on one GPU, residual of the last rep
    n, b = 32768, 1024
    times, _, res = cholesky_run(sf, alg, [dev], n, b, args.streams, args.chol_group, 4, True)
    t = statistics.mean(times[2:])  # two warm-up factorizations (first-use allocations)
    out["cholesky_C3"] = {"n": n, "b": b, "tasks": 5984, "seconds": t, "gflops": alg.flops_cholesky(n) / t / 1e9,
                          "pct_fp64_peak": 100 * alg.flops_cholesky(n) / t / 1e12 / peak_tf,
                          "check": {"cholesky_residual": res, "tol": verify.CHOL_RESIDUAL_TOL,
                                    "pass": res <= verify.CHOL_RESIDUAL_TOL}}
    # C4: particles 2^20 in 256 groups, one evaluation
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, args.streams), trace=False, ordinals=[dev],
                           kernel_timing=True)
    ng, per = 256, 4096
    P = [sf.pinned_empty((4, per)) for _ in range(ng)]
    F = [sf.pinned_empty((4, per)) for _ in range(ng)]
    g = sf.TaskGraph().compute_on(eng)
    alg.insert_fill_particles(g, P, 4)
    g.wait_all()
    ts = []
    for rep in range(3):
        for f in F:
            g.task(sf.write(f), device=sf.ops.zero())
        g.wait_all()
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
    for x in P + F:
        g.flush_to_host(x, keep_device=True)
    g.wait_all()
    pot, force = verify.particle_errors(P, F, verify.sample_particles(ng, per, 48))
    inter = alg.interactions(ng * per)
    dfma_tf = sf.fp64_dfma_peak(dev)
    # mutual kernel: 23 FP64 instructions per unordered pair = 2 ordered interactions
    # (csrc/kernels/particles.cu); FP64-pipe bound = (DFMA peak / 2 flop) instr/s / 11.5
    bound = dfma_tf * 1e12 / 2 / 11.5
    busy = (s1["busy_ns"] - s0["busy_ns"]) * 1e-9
    out["particles_C4"] = {"particles": ng * per, "groups": ng, "tasks": 32896, "seconds": t,
                           "interactions_per_s": inter / t,
                           "gflops_20flop_convention": inter * alg.FLOP_PER_INTERACTION / t / 1e9,
                           "check": {"targets_checked": 48, "pot_rel_err": pot, "force_norm_err": force,
                                     "pass": pot <= verify.POT_REL_TOL and force <= verify.FORCE_NORM_TOL},
                           "roofline": {"bound": "fp64 pipe (DFMA/DMUL/DADD)", "unit": "interactions/s",
                                        "achieved": inter / busy if busy else None,
                                        "peak": bound, "frac": inter / busy / bound if busy else None,
                                        "frac_20flop_convention": (inter * alg.FLOP_PER_INTERACTION / busy / 1e12
                                                                   / dfma_tf) if busy else None,
                                        "dfma_peak_tflops": dfma_tf,
                                        "fp64_instr_per_interaction": 11.5,
                                        "kernel_share_of_step": busy / t,
                                        "launches": s1["timed_groups"] - s0["timed_groups"]}}
    eng.stop()
    # runtime overhead per task: the reference protocol (src/bench.py:67-117)
    T = os.cpu_count() or 4
    out["runtime_overhead"] = {
        "protocol": "reference src/bench.py:67-117: T chains x N tasks, body = D s device spin (no kernel at "
                    "D = 0), deps-1 extra read cells; O_avg = makespan/N - D, O_max = worst end-to-end gap "
                    "in a chain - D (end times = CUDA end events on the host clock), Python insertion cost",
        "runs": overhead_rows(lambda T_, N_, D, mode, deps: overhead_gpu(sf, dev, T_, N_, D, mode, deps),
                              T, args.overhead_n)}
    return out


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
    ordinals = [int(x) for x in args.ordinals.split(",")] if args.ordinals else list(range(ndev))
    if max(ordinals) >= torch.cuda.device_count():
        raise SystemExit(f"bench: {ndev} GPUs requested but only {torch.cuda.device_count()} visible")
    ng, per = 256, 4096
    dfma_tf = sf.fp64_dfma_peak(ordinals[0])
    eng = sf.create_engine(sf.WorkerTeam.of_devices(ndev, args.streams), trace=False, ordinals=ordinals,
                           group_max=args.group)
    P = [sf.pinned_empty((4, per)) for _ in range(ng)]
    F = [sf.pinned_empty((4, per)) for _ in range(ng)]
    g = sf.TaskGraph().compute_on(eng)
    alg.insert_fill_particles(g, P, 4)
    g.wait_all()
    parts = None
    times = []
    clocks = ClockSampler(ordinals)
    for rep in range(args.warmup + args.steps):
        for f in F:
            g.task(sf.write(f), device=sf.ops.zero())
        g.wait_all()
        for d in set(ordinals):
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
    for x in P + F:
        g.flush_to_host(x, keep_device=True)
    g.wait_all()
    pot, force = verify.particle_errors(P, F, verify.sample_particles(ng, per, 48))
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
                   "ordinals": ordinals,
                   "parallelism": "pair tasks in balanced blocks per GPU, per-GPU partial accumulators, "
                                  "dacc reduction (peer pulls)", "l2": "one evaluation per step"},
        "clocks": clk,
        "check": {"targets_checked": 48, "pot_rel_err": pot, "force_norm_err": force,
                  "pass": pot <= verify.POT_REL_TOL and force <= verify.FORCE_NORM_TOL},
        "roofline": {"bound": "fp64 pipe", "achieved": inter / t, "peak": bound, "unit": "interactions/s",
                     "frac": inter / t / bound, "dfma_peak_tflops_per_gpu": dfma_tf},
        "p2p_bytes": sum(s["bytes_p2p_in"] for s in stats),
        "gpu_launches": sum(s["kernel_launches"] for s in stats),
    }
    print(json.dumps(line), flush=True)
    dist.barrier()


def resolve_workload(args, ngpus):
    if args.workload != "auto":
        return args.workload
    return "gemm" if ngpus == 1 else "cholesky"


def main():
    args = parse()
    dist = Dist()
    if args.impl == "reference":
        run_reference(args, dist)
        return
    dist.init("nccl")
    workload = resolve_workload(args, max(args.gpus, dist.world))
    if workload == "cholesky":
        main_cholesky(args, dist)
    elif workload == "particles":
        main_particles(args, dist)
    else:
        if args.gpus > 1 and dist.world == 1:
            raise SystemExit("bench: --workload gemm runs one C2 replica per rank; launch it with torchrun "
                             "for several GPUs (no silent fallback to one GPU)")
        args.n, args.b = args.n or 16384, args.b or 512
        main_gemm(args, dist)
    dist.done()


if __name__ == "__main__":
    main()
