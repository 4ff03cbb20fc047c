"""Parity on the BENCHMARKED paths and at the BASELINE.json sizes (-m gpu).

test_gpu_ops.py checks each op on small shapes; this file closes the gap the
round-1 review named: the kernel configuration the bench spends its time in
(C2: NN b=512, 32-task launch groups, 2 output tiles per persistent CTA, TMA
C-prefetch epilogue, no split-K) is forced and checked, the full-size configs
are verified through size-independent properties (verify.py), and the
reference's own frozen outputs (tests/golden, produced by running the
reference engine) are compared with the native runtime on the GPU.

Tolerances (verify.py):
  GEMM      per-element relative error <= 1e-10; componentwise <= 1e-14
  Cholesky  ||A x - L L^T x|| / (||A||_F ||x||) <= 1e-12 (4 seeded x);
            against the reference's L: max |dL| / max |L| <= 1e-12
  particles potential relative error <= 1e-10; |dF_a| / sum_b |F_ab| <= 1e-12
"""

import os

import numpy as np
import pytest

import paper_2308_15964_b200 as sf
import verify
from paper_2308_15964_b200 import algorithms as alg
from oracle import inputs

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _paths_delta(before):
    now = sf.gemm_paths()
    return {k: now[k] - before[k] for k in now}


def _gemm_engine(streams=32, group=32):
    return sf.create_engine(sf.WorkerTeam.of_devices(1, streams), scheduler="prio", trace=False, group_max=group)


def test_headline_dgemm_path_full_product():
    """Tiled 3072/512 (36 C chains) inserted behind the gate: the first k-wave is
    36 ready same-shape NN tasks -> a launch group of 32 tasks = 512 output tiles
    -> 2 tiles per persistent CTA with the C-prefetch epilogue and no split-K
    (the C2 bench configuration).  The whole product is compared with numpy."""
    n, b = 3072, 512
    eng = _gemm_engine()
    try:
        A, B, C = (alg.TiledMatrix(n, b) for _ in range(3))
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_fill_uniform(g, A, 1)
        alg.insert_fill_uniform(g, B, 2)
        alg.insert_zero(g, C)
        assert g.wait_all(timeout=120)
        before = sf.gemm_paths()
        with g.gated():
            alg.insert_gemm(g, A, B, C)
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=120)
        d = _paths_delta(before)
        assert d["cpref_multi_tile"] >= 1, d  # the headline configuration ran (first k-wave)
        Ad, Bd, Cd = A.to_dense(), B.to_dense(), C.to_dense()
        assert np.array_equal(Ad, inputs.uniform_tile(1, 0, 0, n, n, n))
        want = Ad @ Bd
        rel = np.abs(Cd - want) / np.abs(want)
        assert rel.max() <= verify.GEMM_REL_TOL, rel.max()
    finally:
        eng.stop()


def test_headline_dgemm_path_repeated_steps_accumulate():
    """Three C += A B steps through the persistent 2-tile loop: the C-prefetch
    buffer is handed between consecutive tiles of one CTA (cempty parity) every
    launch; C = 3 A B on sampled tiles."""
    n, b = 4096, 512
    eng = _gemm_engine()
    try:
        A, B, C = (alg.TiledMatrix(n, b) for _ in range(3))
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_fill_uniform(g, A, 5)
        alg.insert_fill_uniform(g, B, 6)
        alg.insert_zero(g, C)
        assert g.wait_all(timeout=120)
        before = sf.gemm_paths()
        for _ in range(3):
            alg.insert_gemm(g, A, B, C)
        g.flush_all(keep_device=True)
        assert g.wait_all(timeout=180)
        d = _paths_delta(before)
        assert d["cpref_multi_tile"] >= 1 and d["tasks"] == 3 * (n // b) ** 3, d
        rel, comp = verify.gemm_tile_errors(C.tiles, A.tiles, B.tiles, verify.sample_tiles(n // b, 6), mult=3.0)
        assert rel <= verify.GEMM_REL_TOL and comp <= verify.GEMM_COMPONENTWISE_TOL, (rel, comp)
    finally:
        eng.stop()


def test_c2_full_size_sampled_tiles():
    """C2 itself (16384 / 512, 32,768 tasks) with the bench's engine settings;
    sampled C tiles against numpy."""
    n, b = 16384, 512
    eng = _gemm_engine()
    try:
        A, B, C = (alg.TiledMatrix(n, b) for _ in range(3))
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_fill_uniform(g, A, 1)
        alg.insert_fill_uniform(g, B, 2)
        alg.insert_zero(g, C)
        assert g.wait_all(timeout=120)
        before = sf.gemm_paths()
        alg.insert_gemm(g, A, B, C)
        g.flush_all(keep_device=True)
        assert g.wait_all(timeout=300)
        d = _paths_delta(before)
        assert d["tasks"] == (n // b) ** 3 and d["cpref_multi_tile"] >= 1, d
        rel, comp = verify.gemm_tile_errors(C.tiles, A.tiles, B.tiles, verify.sample_tiles(n // b, 4, seed=3))
        assert rel <= verify.GEMM_REL_TOL and comp <= verify.GEMM_COMPONENTWISE_TOL, (rel, comp)
    finally:
        eng.stop()


def test_c1_matches_reference_engine_golden():
    """C1 (DGEMM 2048/256) through the drop-in API against the values the
    REFERENCE engine produced (tests/golden/numerics.npz, make_golden.py)."""
    gold = np.load(os.path.join(GOLD, "numerics.npz"))
    n, b = 2048, 256
    eng = _gemm_engine(8, 32)
    try:
        A, B, C = (alg.TiledMatrix(n, b) for _ in range(3))
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_fill_uniform(g, A, 1)
        alg.insert_fill_uniform(g, B, 2)
        alg.insert_zero(g, C)
        alg.insert_gemm(g, A, B, C)
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=120)
    finally:
        eng.stop()
    Cd = C.to_dense()
    for got, want in ((Cd[::17, ::19], gold["gemm_C_sample"]), (Cd.sum(axis=1), gold["gemm_C_rowsum"]),
                      (Cd.sum(axis=0), gold["gemm_C_colsum"])):
        rel = np.abs(got - want) / np.abs(want)
        assert rel.max() <= verify.GEMM_REL_TOL, rel.max()


def test_cholesky_1024_128_matches_reference_engine_golden():
    gold = np.load(os.path.join(GOLD, "numerics.npz"))
    n, b = 1024, 128
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 8), scheduler="prio", device_memory=1 << 30)
    try:
        M = alg.TiledMatrix(n, b, lower=True)
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_fill_spd(g, M, 3)
        alg.insert_cholesky(g, M)
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=120)
    finally:
        eng.stop()
    L = M.to_dense(lower_only=True)
    Lg = gold["chol_L"]
    got = L[np.tril_indices(n)][::7]
    assert np.abs(got - Lg).max() / np.abs(Lg).max() <= 1e-12
    assert np.abs(L.sum(axis=1) - gold["chol_L_rowsum"]).max() / np.abs(gold["chol_L_rowsum"]).max() <= 1e-12


def test_particles_8x256_match_reference_engine_golden():
    gold = np.load(os.path.join(GOLD, "numerics.npz"))["particles_F"]
    ng, per = 8, 256
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 4), device_memory=1 << 30)
    try:
        P = [sf.pinned_empty((4, per)) for _ in range(ng)]
        F = [sf.pinned_zeros((4, per)) for _ in range(ng)]
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_fill_particles(g, P, 4)
        alg.insert_particles(g, P, F)
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=120)
    finally:
        eng.stop()
    for gi in range(ng):
        w = gold[gi]
        assert (np.abs(F[gi][3] - w[3]) / np.abs(w[3])).max() <= verify.POT_REL_TOL
        assert np.abs(F[gi][:3] - w[:3]).max() <= 1e-11 * np.abs(w[:3]).max()


def test_c3_full_size_randomized_residual():
    """C3: Cholesky 32768 / 1024 (5,984 tasks) with the bench's settings; the
    randomized residual on 4 seeded vectors."""
    n, b = 32768, 1024
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 32), scheduler="prio", trace=False, group_max=8)
    try:
        M = alg.TiledMatrix(n, b, lower=True)
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_fill_spd(g, M, 3)
        g.flush_all(keep_device=True)
        assert g.wait_all(timeout=120)
        A = {ij: t.copy() for ij, t in M.tiles.items()}
        assert np.array_equal(A[(3, 1)], inputs.spd_tile(3, 3 * b, b, b, b, n))
        alg.insert_cholesky(g, M)
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=300)
    finally:
        eng.stop()
    res = verify.cholesky_residual(A, M.tiles, n, b)
    assert res <= verify.CHOL_RESIDUAL_TOL, res


def test_c4_full_size_sampled_particles():
    """C4: 2^20 particles in 256 groups (32,896 commutative tasks); 48 sampled
    targets against all 2^20 sources."""
    ng, per = 256, 4096
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 32), trace=False)
    try:
        P = [sf.pinned_empty((4, per)) for _ in range(ng)]
        F = [sf.pinned_zeros((4, per)) for _ in range(ng)]
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_fill_particles(g, P, 4)
        alg.insert_particles(g, P, F)
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=300)
    finally:
        eng.stop()
    pot, force = verify.particle_errors(P, F, verify.sample_particles(ng, per, 48))
    assert pot <= verify.POT_REL_TOL and force <= verify.FORCE_NORM_TOL, (pot, force)


def test_c5_shape_trace_nt64_is_bit_exact_with_the_reference():
    """Cholesky nt = 64 (the C5 graph: 45,760 tasks, 131,040 edges) on the native
    runtime with the real tile kernels (tiles of 64): edges and the deterministic
    one-stream FIFO pop order equal the reference engine's (tile_graphs.npz)."""
    gold = np.load(os.path.join(GOLD, "tile_graphs.npz"))
    nt, b = 64, 64
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 1), scheduler=None, device_memory=1 << 30, group_max=1)
    try:
        M = alg.TiledMatrix(nt * b, b, lower=True)
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_fill_spd(g, M, 3)
        assert g.wait_all(timeout=60)
        with g.gated():
            tids = alg.insert_cholesky(g, M, priorities=False).tolist()
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=600)
        index = {t: i for i, t in enumerate(tids)}
        edges = sorted({(index[s], index[d]) for s, d, _ in g.edges() if s in index and d in index})
        assert len(edges) == 131040
        assert edges == sorted(map(tuple, gold["cholesky_nt64_edges"].tolist()))
        pops = [index[e[3]] for e in g.trace.export_events() if e[0] == "Pop" and e[3] in index]
        assert pops == gold["cholesky_nt64_pop"].tolist()
        A0 = {ij: inputs.spd_tile(3, ij[0] * b, ij[1] * b, b, b, nt * b) for ij in M.tiles}
        assert verify.cholesky_residual(A0, M.tiles, nt * b, b) <= verify.CHOL_RESIDUAL_TOL
    finally:
        eng.stop()


def test_c4_shape_trace_g256_is_bit_exact_with_the_reference():
    """The particle graph with 256 groups (32,896 tasks, all commutative): no
    edges, and the one-stream FIFO pop order equals the reference's."""
    gold = np.load(os.path.join(GOLD, "tile_graphs.npz"))
    ng, per = 256, 32
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 1), scheduler=None, device_memory=1 << 30, group_max=1)
    try:
        P = [sf.pinned_empty((4, per)) for _ in range(ng)]
        F = [sf.pinned_zeros((4, per)) for _ in range(ng)]
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_fill_particles(g, P, 4)
        assert g.wait_all(timeout=60)
        with g.gated():
            tids = alg.insert_particles(g, P, F).tolist()
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=600)
        index = {t: i for i, t in enumerate(tids)}
        edges = sorted({(index[s], index[d]) for s, d, _ in g.edges() if s in index and d in index})
        assert edges == sorted(map(tuple, gold["particles_g256_edges"].reshape(-1, 2).tolist()))
        pops = [index[e[3]] for e in g.trace.export_events() if e[0] == "Pop" and e[3] in index]
        assert pops == gold["particles_g256_pop"].tolist()
        pot, force = verify.particle_errors(P, F, verify.sample_particles(ng, per, 16))
        assert pot <= verify.POT_REL_TOL and force <= verify.FORCE_NORM_TOL, (pot, force)
    finally:
        eng.stop()
