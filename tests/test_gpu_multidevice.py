"""Multi-device execution on real CUDA: the runtime drives two LOGICAL devices
mapped onto one physical B200 (separate arenas, streams, executors and
completion threads; cudaMemcpyPeerAsync between them degenerates to a device
copy).  This exercises placement, peer pulls, cross-device event waits and
invalidation with the real backend even on a single-GPU box."""

import os

import numpy as np
import pytest

import paper_2308_15964_b200 as sf
from paper_2308_15964_b200 import algorithms as alg
from oracle import inputs, programs

pytestmark = pytest.mark.gpu


def two_device_engine(streams=4):
    return sf.create_engine(sf.WorkerTeam.of_devices(2, streams), scheduler="prio", device_memory=2 << 30,
                            ordinals=[0, 0])


def test_block_cyclic_cholesky_on_two_devices():
    n, b = 2048, 256
    objs = programs.cholesky_operands(n, b)
    want = {k: v.copy() for k, v in objs.items()}
    programs.run_on_oracle(programs.cholesky_program(n // b), want, workers=4).stop()
    eng = two_device_engine()
    try:
        M = alg.TiledMatrix(n, b, lower=True)
        for ij, t in M.tiles.items():
            t[...] = objs[("A",) + ij]
        g = sf.TaskGraph().compute_on(eng)
        alg.block_cyclic(g, M, *alg.grid_shape(2))
        alg.insert_cholesky(g, M)
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=120)
        s0, s1 = eng.stats(0), eng.stats(1)
        assert s0["tasks_executed"] > 0 and s1["tasks_executed"] > 0
        assert s0["bytes_p2p_in"] + s1["bytes_p2p_in"] > 0  # panels moved device-to-device
        L = M.to_dense(lower_only=True)
        Lw = programs.assemble_lower(want, n, b)
        assert np.abs(L - Lw).max() / np.abs(Lw).max() <= 1e-12
        assert eng.violations() == 0
    finally:
        eng.stop()


def test_random_programs_on_two_devices():
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "random_programs.json")) as fh:
        progs = json.load(fh)
    mode = {"read": sf.read, "write": sf.write, "atomic": sf.atomic_write, "commute": sf.commutative_write,
            "maybe": sf.maybe_write}
    eng = two_device_engine(2)
    try:
        for p in progs[:60]:
            g = sf.TaskGraph().compute_on(eng)
            cells = [sf.Cell(i + 1) for i in range(p["n_cells"])]
            for m, target, reads, a, b in p["tasks"]:
                acc = [mode[m](cells[target])] + [sf.read(cells[r]) for r in reads]
                g.task(*acc, device=sf.ops.cell(m, a, b))
            for c in cells:
                g.flush_to_host(c)
            assert g.wait_all(timeout=60)
            assert [c.value for c in cells] == p["sequential"]
    finally:
        eng.stop()


@pytest.mark.parametrize("ndev", [2, 3])
def test_particles_with_per_device_partials(ndev):
    """SURVEY.md §8e for C4: pair tasks dealt to the devices, private per-device
    accumulators, one dacc reduction per group (peer pulls) -- same result as the
    oracle within the particle tolerances."""
    ng, per = 6, 512
    objs = programs.particle_operands(ng, per)
    want = {k: v.copy() for k, v in objs.items()}
    programs.run_on_oracle(programs.particles_program(ng), want, workers=4)
    eng = sf.create_engine(sf.WorkerTeam.of_devices(ndev, 3), device_memory=1 << 30, ordinals=[0] * ndev)
    try:
        P = [sf.pinned_empty((4, per)) for _ in range(ng)]
        F = [sf.pinned_zeros((4, per)) for _ in range(ng)]
        for g in range(ng):
            P[g][...] = objs[("P", g)]
        gr = sf.TaskGraph().compute_on(eng)
        parts = alg.insert_particles(gr, P, F)
        assert parts is not None and len(parts) == ndev - 1
        gr.flush_all(keep_device=False)
        assert gr.wait_all(timeout=120)
        assert all(eng.stats(d)["tasks_executed"] > 0 for d in range(ndev))
        assert sum(eng.stats(d)["bytes_p2p_in"] for d in range(ndev)) > 0
        for g in range(ng):
            w = want[("F", g)]
            assert (np.abs(F[g][3] - w[3]) / np.abs(w[3])).max() <= 1e-10
            assert np.abs(F[g][:3] - w[:3]).max() <= 1e-11 * np.abs(w[:3]).max()
    finally:
        eng.stop()


def test_real_cholesky_trace_is_bit_exact_with_the_reference():
    """The dependency trace of the REAL GPU Cholesky (tile kernels on the B200, 32x32
    tiles of 64) equals the reference's: the 16,368 dot edges and, in the
    deterministic mode (1 GPU, 1 stream, FIFO, no grouping, gated insertion), the
    one-worker pop order frozen from the reference engine (tests/golden)."""
    import os

    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "tile_graphs.npz"))
    nt, b = 32, 64
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 1), scheduler=None, device_memory=1 << 30, group_max=1)
    try:
        M = alg.TiledMatrix(nt * b, b, lower=True)
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_fill_spd(g, M, 3)  # same graph: the filled tiles stay resident (device-dirty)
        assert g.wait_all(timeout=60)
        with g.gated():
            tids = alg.insert_cholesky(g, M, priorities=False).tolist()
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=120)
        index = {t: i for i, t in enumerate(tids)}
        edges = sorted({(index[s], index[d]) for s, d, _ in g.edges() if s in index and d in index})
        assert len(edges) == 16368
        assert edges == sorted(map(tuple, gold["cholesky_nt32_edges"].tolist()))
        pops = [index[e[3]] for e in g.trace.export_events() if e[0] == "Pop" and e[3] in index]
        assert pops == gold["cholesky_nt32_pop"].tolist()
        # and the factor is right
        A0 = np.zeros((nt * b, nt * b))
        for (i, j), _ in M.tiles.items():
            A0[i * b:(i + 1) * b, j * b:(j + 1) * b] = inputs.spd_tile(3, i * b, j * b, b, b, nt * b)
        A0 = np.tril(A0) + np.tril(A0, -1).T
        L = M.to_dense(lower_only=True)
        assert np.linalg.norm(A0 - L @ L.T) / np.linalg.norm(A0) <= 1e-12
    finally:
        eng.stop()


def test_real_gemm_trace_is_bit_exact_with_the_reference():
    """Same for the tiled DGEMM (C1 shape: 8x8 tiles, here of 64): 448 edges and the
    reference's one-worker FIFO pop order, with the real DMMA tile kernels."""
    import os

    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "tile_graphs.npz"))
    nt, b = 8, 64
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 1), scheduler=None, device_memory=1 << 30, group_max=1)
    try:
        A, B, C = (alg.TiledMatrix(nt * b, b) for _ in range(3))
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_fill_uniform(g, A, 1)
        alg.insert_fill_uniform(g, B, 2)
        alg.insert_zero(g, C)
        assert g.wait_all(timeout=60)
        with g.gated():
            tids = alg.insert_gemm(g, A, B, C).tolist()
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=60)
        index = {t: i for i, t in enumerate(tids)}
        edges = sorted({(index[s], index[d]) for s, d, _ in g.edges() if s in index and d in index})
        assert edges == sorted(map(tuple, gold["gemm_nt8_edges"].tolist()))
        pops = [index[e[3]] for e in g.trace.export_events() if e[0] == "Pop" and e[3] in index]
        assert pops == gold["gemm_nt8_pop"].tolist()
        Ad = np.vstack([np.hstack([inputs.uniform_tile(1, i * b, j * b, b, b, nt * b) for j in range(nt)])
                        for i in range(nt)])
        Bd = np.vstack([np.hstack([inputs.uniform_tile(2, i * b, j * b, b, b, nt * b) for j in range(nt)])
                        for i in range(nt)])
        want = Ad @ Bd
        assert (np.abs(C.to_dense() - want) / np.abs(want)).max() <= 1e-10
    finally:
        eng.stop()


@pytest.mark.parametrize("streams", [1, 2, 4])
def test_random_programs_through_a_tiny_arena_on_the_gpu(streams):
    """The reference's random programs (every access mode) on real CUDA streams
    through an arena of four 64-byte slots: most accesses evict, dirty cells are
    written back and re-staged while other streams run, and the executor often
    has to wait for a completion before it can plan (this found a missed
    wake-up that hung the engine).  Values equal the sequential execution
    frozen from the reference."""
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "random_programs.json")) as fh:
        progs = json.load(fh)
    mode = {"read": sf.read, "write": sf.write, "atomic": sf.atomic_write, "commute": sf.commutative_write,
            "maybe": sf.maybe_write}
    widest = max(1 + len(t[2]) for q in progs[:60] for t in q["tasks"])
    assert widest <= 4  # the CUDA arena is at least 256 bytes: 4 slots of 64
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, streams), device_memory=256, arena_align=64)
    try:
        for p in progs[:60]:
            g = sf.TaskGraph().compute_on(eng)
            cells = [sf.Cell(i + 1) for i in range(p["n_cells"])]
            for m, target, reads, a, b in p["tasks"]:
                acc = [mode[m](cells[target])] + [sf.read(cells[r]) for r in reads]
                g.task(*acc, device=sf.ops.cell(m, a, b))
            for c in cells:
                g.flush_to_host(c)
            assert g.wait_all(timeout=60)
            assert [c.value for c in cells] == p["sequential"]
        assert eng.stats(0)["evictions"] > 0
    finally:
        eng.stop()


@pytest.mark.parametrize("ndev,streams", [(2, 2), (3, 1)])
def test_random_programs_across_devices_through_tiny_arenas(ndev, streams):
    """Logical devices with four 64-byte slots each: peer pulls, invalidations
    (zombie blocks pinned by another device's task), evictions and write-backs
    interleave; the executor must wait for completions on ANY device before
    declaring the arena exhausted (this found a spurious StagingError).  Values
    equal the reference's sequential execution for all 120 programs."""
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "random_programs.json")) as fh:
        progs = json.load(fh)
    mode = {"read": sf.read, "write": sf.write, "atomic": sf.atomic_write, "commute": sf.commutative_write,
            "maybe": sf.maybe_write}
    eng = sf.create_engine(sf.WorkerTeam.of_devices(ndev, streams), device_memory=256, arena_align=64,
                           ordinals=[0] * ndev)
    try:
        for p in progs:
            g = sf.TaskGraph().compute_on(eng)
            cells = [sf.Cell(i + 1) for i in range(p["n_cells"])]
            for m, target, reads, a, b in p["tasks"]:
                acc = [mode[m](cells[target])] + [sf.read(cells[r]) for r in reads]
                g.task(*acc, device=sf.ops.cell(m, a, b))
            for c in cells:
                g.flush_to_host(c)
            assert g.wait_all(timeout=60)
            assert [c.value for c in cells] == p["sequential"]
        assert sum(eng.stats(d)["evictions"] for d in range(ndev)) > 0
        assert sum(eng.stats(d)["bytes_p2p_in"] for d in range(ndev)) > 0
    finally:
        eng.stop()


def test_tile_cache_stress_with_requeued_groups():
    """Regression test for the write-back race: a Cholesky through a 13-slot tile
    cache with launch groups that run out of space mid-group (the staging-aware
    group limit switched off, so requeued members re-plan on other streams over
    ranges still being written back).  Every factor must be exact."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SFX_GROUP_NO_STAGE_LIMIT="1", GM="8")
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "arena_stress.py"), "12", "full", "4", "1"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "wrong factors: 0 of 12" in r.stdout, r.stdout[-2000:]
