"""Generate golden fixtures by running the REAL reference ``seqflow`` in this container.

The reference is pure Python, importable from
/root/reference/pkg/src; it does not exist on the GPU box, so its outputs are
frozen here as small fixtures that the tests (CPU and GPU) compare against.

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_golden.py

Fixtures:
  random_programs.json  reference random programs (tests/conftest.py:49-60):
                        sequential values, successor edges and one-worker pop
                        order under gated insertion (tests/conftest.py:184-203)
  tile_graphs.npz       the north-star tile graphs (C1 DGEMM nt=8, Cholesky
                        nt=8/32/64, particles 16/256 groups) inserted into the
                        reference engine (1 worker, gated, no-op bodies): edges
                        and pop order as insertion indices
  lru.json              resident sets of the reference arena (src/device.py
                        DeviceDomain, via tests/test_device.py:_touch) for the
                        criterion-5 (seed 5) and test_device (seed 20240) sequences
  numerics.npz          tile workloads executed BY THE REFERENCE ENGINE with the
                        oracle's numpy bodies: C1 DGEMM 2048/256, Cholesky
                        1024/128, particles 8 x 256
"""

from __future__ import annotations

import json
import os
import random
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
for p in ("/root/reference/pkg/src", "/root/reference/pkg/tests"):
    if p not in sys.path:
        sys.path.insert(0, p)

import seqflow as sf  # noqa: E402  (the reference)
from conftest import (  # noqa: E402  (the reference's test fixtures)
    parse_dot,
    random_program,
    run_gated_program,
    sequential_oracle,
    static_successor_edges,
)
from seqflow.device import DeviceDomain  # noqa: E402
from test_device import ReferenceLRU, _FakeHandle, _touch  # noqa: E402

from oracle import bodies, programs  # noqa: E402
from oracle.stf import COMMUTE, MAYBE, READ, WRITE, ATOMIC  # noqa: E402

_MODE = {READ: sf.read, WRITE: sf.write, COMMUTE: sf.commutative_write, MAYBE: sf.maybe_write,
         ATOMIC: sf.atomic_write}


def _pop_indices(graph, tids):
    index = {t: i for i, t in enumerate(tids)}
    return [index[e[3]] for e in graph.trace.export_events() if e[0] == "Pop" and e[3] in index]


def gen_random_programs():
    out = []
    eng = sf.create_engine(sf.WorkerTeam.of_host_workers(1))
    try:
        for seed, count, max_tasks, max_cells in ((8, 60, 40, 8), (1, 60, 64, 16)):
            rng = random.Random(seed)
            for _ in range(count):
                n_cells, tasks = random_program(rng, max_tasks=max_tasks, max_cells=max_cells)
                g, tids, values = run_gated_program(eng, n_cells, tasks)
                _, edges = parse_dot(sf.generate_dot(g))
                index = {t: i for i, t in enumerate(tids)}
                eidx = sorted((index[a], index[b]) for a, b in edges if a in index and b in index)
                assert set(eidx) == static_successor_edges(n_cells, tasks)
                out.append({
                    "seed": seed,
                    "n_cells": n_cells,
                    "tasks": [[t.mode, t.target, list(t.reads), t.a, t.b] for t in tasks],
                    "values": values,
                    "sequential": sequential_oracle(n_cells, tasks),
                    "edges": eidx,
                    "pop_order": _pop_indices(g, tids),
                })
    finally:
        eng.stop()
    with open(os.path.join(HERE, "random_programs.json"), "w") as fh:
        json.dump(out, fh)
    print("random_programs:", len(out))


def _run_reference_gated(prog):
    """Insert a tile program into the reference engine behind a gate; no-op bodies."""
    objs = {}
    eng = sf.create_engine(sf.WorkerTeam.of_host_workers(1))
    try:
        g = sf.TaskGraph().compute_on(eng)
        gate = threading.Event()
        g.task(sf.read(sf.Cell(0)), host=lambda c: gate.wait(600), name="gate")
        tids = []
        for kind, acc, prio in prog:
            specs = []
            for mode, key in acc:
                if key not in objs:
                    objs[key] = sf.Cell(0)
                specs.append(_MODE[mode](objs[key]))
            tids.append(g.task(*specs, host=lambda *a: None, name=kind).task_id)
        gate.set()
        assert g.wait_all(timeout=600)
        index = {t: i for i, t in enumerate(tids)}
        _, edges = parse_dot(sf.generate_dot(g))
        eidx = np.array(sorted((index[a], index[b]) for a, b in edges if a in index and b in index),
                        dtype=np.int32).reshape(-1, 2)
        pop = np.array(_pop_indices(g, tids), dtype=np.int32)
    finally:
        eng.stop()
    return eidx, pop


def gen_tile_graphs():
    graphs = {
        "gemm_nt8": programs.gemm_program(8),
        "cholesky_nt8": programs.cholesky_program(8),
        "cholesky_nt32": programs.cholesky_program(32),
        "cholesky_nt64": programs.cholesky_program(64),
        "particles_g16": programs.particles_program(16),
        "particles_g256": programs.particles_program(256),
    }
    out = {}
    for name, prog in graphs.items():
        t0 = time.time()
        edges, pop = _run_reference_gated(prog)
        out[f"{name}_edges"] = edges
        out[f"{name}_pop"] = pop
        out[f"{name}_ntasks"] = np.array([len(prog)], dtype=np.int64)
        print(f"tile graph {name}: {len(prog)} tasks, {len(edges)} edges ({time.time() - t0:.1f} s)")
    np.savez_compressed(os.path.join(HERE, "tile_graphs.npz"), **out)


def gen_lru():
    cases = []
    for seed, trials, steps, size, nh, slots in ((5, 200, 80, 32, 10, (2, 6)), (20240, 30, 120, 64, 12, (2, 6))):
        rng = random.Random(seed)
        for _ in range(trials):
            n_slots = rng.randint(*slots)
            domain = DeviceDomain(0, n_slots * size)
            ref = ReferenceLRU(n_slots * size)
            handles = [_FakeHandle(h, bytearray([h % 256] * size)) for h in range(nh)]
            seq, resident = [], []
            for _ in range(steps):
                h = rng.randrange(nh)
                _touch(domain, handles[h])
                ref.access(h, size)
                assert set(domain.arena.blocks) == set(ref.blocks)
                seq.append(h)
                resident.append(sorted(domain.arena.blocks))
            cases.append({"seed": seed, "capacity": n_slots * size, "size": size, "seq": seq, "resident": resident})
    with open(os.path.join(HERE, "lru.json"), "w") as fh:
        json.dump(cases, fh)
    print("lru cases:", len(cases))


def _run_reference_numeric(prog, objs, workers):
    eng = sf.create_engine(sf.WorkerTeam.of_host_workers(workers))
    try:
        g = sf.TaskGraph().compute_on(eng)
        for kind, acc, prio in prog:
            g.task(*[_MODE[m](objs[k]) for m, k in acc], host=bodies.BODIES[kind], priority=prio)
        assert g.wait_all(timeout=600)
    finally:
        eng.stop()


def gen_numerics():
    from threadpoolctl import threadpool_limits

    out = {}
    with threadpool_limits(1):
        # C1: DGEMM 2048 / 256 ("oracle run")
        n, b = 2048, 256
        objs = programs.gemm_operands(n, b)
        t0 = time.time()
        _run_reference_numeric(programs.gemm_program(n // b), objs, 8)
        out["gemm_seconds"] = np.array([time.time() - t0])
        C = np.block([[objs[("C", i, j)] for j in range(n // b)] for i in range(n // b)])
        out["gemm_C_rowsum"] = C.sum(axis=1)
        out["gemm_C_colsum"] = C.sum(axis=0)
        out["gemm_C_sample"] = C[::17, ::19].copy()
        # Cholesky 1024 / 128
        n, b = 1024, 128
        objs = programs.cholesky_operands(n, b)
        _run_reference_numeric(programs.cholesky_program(n // b), objs, 8)
        L = programs.assemble_lower(objs, n, b)
        out["chol_L"] = L[np.tril_indices(n)][::7].copy()
        out["chol_L_rowsum"] = L.sum(axis=1)
        # particles 8 x 256
        ng, per = 8, 256
        objs = programs.particle_operands(ng, per)
        _run_reference_numeric(programs.particles_program(ng), objs, 8)
        out["particles_F"] = np.stack([objs[("F", g)] for g in range(ng)])
    np.savez_compressed(os.path.join(HERE, "numerics.npz"), **out)
    print("numerics done; C1 via reference engine:", float(out["gemm_seconds"][0]), "s")


if __name__ == "__main__":
    which = set(sys.argv[1:]) or {"random", "tiles", "lru", "numerics"}
    if "random" in which:
        gen_random_programs()
    if "lru" in which:
        gen_lru()
    if "numerics" in which:
        gen_numerics()
    if "tiles" in which:
        gen_tile_graphs()
