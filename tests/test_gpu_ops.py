"""GPU parity of the tile ops and the tiled workloads against the CPU oracle.

Tolerances (BASELINE.json north_star / SURVEY.md §8d):
  GEMM       per-element relative error <= 1e-10 (uniform inputs, no cancellation)
  Cholesky   ||A - L L^T||_F / ||A||_F <= 1e-12, and L within 1e-10 of the oracle's L
  TRSM       relative residual ||X L^T - B|| / (||L|| ||X||) <= 1e-13, normwise vs oracle <= 1e-12
  particles  per-particle potential rel err <= 1e-10; |dF_a| / sum_b |F_ab| <= 1e-12
"""

import numpy as np
import pytest

import paper_2308_15964_b200 as sf
from paper_2308_15964_b200 import algorithms as alg
from oracle import bodies, inputs, programs

pytestmark = pytest.mark.gpu


def _run(eng, fn):
    g = sf.TaskGraph().compute_on(eng)
    fn(g)
    g.flush_all(keep_device=False)
    assert g.wait_all(timeout=120)
    return g


@pytest.mark.parametrize("b,trans_b", [(256, False), (256, True), (512, True), (320, False)])
def test_dgemm_tile(gpu_engine, b, trans_b):
    A = inputs.uniform_tile(11, 0, 0, b, b, b)
    B = inputs.uniform_tile(12, 0, 0, b, b, b)
    C = inputs.uniform_tile(13, 0, 0, b, b, b)
    want = C + A @ (B.T if trans_b else B)
    _run(gpu_engine, lambda g: g.task(sf.read(A), sf.read(B), sf.write(C), device=sf.ops.dgemm(1.0, 1.0, trans_b)))
    rel = np.abs(C - want) / np.abs(want)
    assert rel.max() <= 1e-10, rel.max()


def test_dsyrk_tile_lower_only(gpu_engine):
    b = 512
    A = inputs.uniform_tile(21, 0, 0, b, b, b)
    C0 = inputs.uniform_tile(22, 0, 0, b, b, b) + b
    C = C0.copy()
    want = C0.copy()
    bodies.syrk_sub(A, want)
    _run(gpu_engine, lambda g: g.task(sf.read(A), sf.write(C), device=sf.ops.syrk_sub))
    il = np.tril_indices(b)
    iu = np.triu_indices(b, 1)
    assert np.array_equal(C[iu], C0[iu])  # upper triangle untouched
    assert (np.abs(C[il] - want[il]) / np.abs(want[il])).max() <= 1e-10


@pytest.mark.parametrize("b", [256, 1024])
def test_dtrsm_tile(gpu_engine, b):
    S = inputs.spd_tile(31, 0, 0, b, b, b)
    L = np.linalg.cholesky(S)
    B = inputs.uniform_tile(32, 0, 0, b, b, b)
    X = B.copy()
    _run(gpu_engine, lambda g: g.task(sf.read(L), sf.write(X), device=sf.ops.trsm))
    want = B.copy()
    bodies.trsm(L, want)
    res = np.linalg.norm(X @ L.T - B) / (np.linalg.norm(L) * np.linalg.norm(X))
    assert res <= 1e-13, res
    # per-element relative error is ill-posed for a solve (entries cancel); normwise instead
    assert np.linalg.norm(X - want) / np.linalg.norm(want) <= 1e-12


@pytest.mark.parametrize("b", [64, 256, 1024])
def test_dpotrf_tile(gpu_engine, b):
    A0 = inputs.spd_tile(41, 0, 0, b, b, b)
    A = A0.copy()
    _run(gpu_engine, lambda g: g.task(sf.write(A), device=sf.ops.potrf))
    L = np.tril(A)
    assert np.linalg.norm(A0 - L @ L.T) / np.linalg.norm(A0) <= 1e-12
    iu = np.triu_indices(b, 1)
    assert np.array_equal(A[iu], A0[iu])  # LAPACK 'L' semantics: upper untouched
    want = A0.copy()
    bodies.potrf(want)
    assert (np.abs(L - np.tril(want)).max() / np.abs(want).max()) <= 1e-12


def test_generators_bit_identical(gpu_engine):
    n, b = 512, 256
    U = alg.TiledMatrix(n, b)
    S = alg.TiledMatrix(n, b, lower=True)
    P = [sf.pinned_empty((4, 128)) for _ in range(3)]
    def fill(g):
        alg.insert_fill_uniform(g, U, 7)
        alg.insert_fill_spd(g, S, 3)
        alg.insert_fill_particles(g, P, 4)
    _run(gpu_engine, fill)
    for (i, j), t in U.tiles.items():
        assert np.array_equal(t, inputs.uniform_tile(7, i * b, j * b, b, b, n))
    for (i, j), t in S.tiles.items():
        assert np.array_equal(t, inputs.spd_tile(3, i * b, j * b, b, b, n))
    for g, p in enumerate(P):
        assert np.array_equal(p, inputs.particles(4, g * 128, 128))


def test_tiled_gemm_matches_oracle(gpu_engine):
    n, b = 1024, 256
    objs = programs.gemm_operands(n, b)
    want = {k: v.copy() for k, v in objs.items()}
    programs.run_on_oracle(programs.gemm_program(n // b), want, workers=4)
    A, B, C = (alg.TiledMatrix(n, b) for _ in range(3))
    for (i, j) in A.tiles:
        A[i, j][...] = objs[("A", i, j)]
        B[i, j][...] = objs[("B", i, j)]
        C[i, j][...] = 0.0
    _run(gpu_engine, lambda g: alg.insert_gemm(g, A, B, C))
    for (i, j), t in C.tiles.items():
        w = want[("C", i, j)]
        assert (np.abs(t - w) / np.abs(w)).max() <= 1e-10


def test_tiled_cholesky_matches_oracle(gpu_engine):
    n, b = 2048, 256
    objs = programs.cholesky_operands(n, b)
    A0 = programs.assemble_lower(objs, n, b)
    A0 = A0 + np.tril(A0, -1).T
    want = {k: v.copy() for k, v in objs.items()}
    programs.run_on_oracle(programs.cholesky_program(n // b), want, workers=4)
    M = alg.TiledMatrix(n, b, lower=True)
    for ij, t in M.tiles.items():
        t[...] = objs[("A",) + ij]
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 8), scheduler="prio", device_memory=4 << 30)
    try:
        _run(eng, lambda g: alg.insert_cholesky(g, M))
    finally:
        eng.stop()
    L = M.to_dense(lower_only=True)
    assert np.linalg.norm(A0 - L @ L.T) / np.linalg.norm(A0) <= 1e-12
    Lw = programs.assemble_lower(want, n, b)
    assert np.abs(L - Lw).max() / np.abs(Lw).max() <= 1e-12


def test_particles_match_oracle(gpu_engine):
    ng, per = 6, 512
    objs = programs.particle_operands(ng, per)
    want = {k: v.copy() for k, v in objs.items()}
    programs.run_on_oracle(programs.particles_program(ng), want, workers=4)
    P = [sf.pinned_empty((4, per)) for _ in range(ng)]
    F = [sf.pinned_zeros((4, per)) for _ in range(ng)]
    for g in range(ng):
        P[g][...] = objs[("P", g)]
    _run(gpu_engine, lambda g: alg.insert_particles(g, P, F))
    for g in range(ng):
        w = want[("F", g)]
        got = F[g]
        pot_rel = np.abs(got[3] - w[3]) / np.abs(w[3])
        assert pot_rel.max() <= 1e-10, pot_rel.max()
        # normalised force error: |dF_a| / sum_b |F_ab|  (sum_b |F_ab| bounded below by |F_a|)
        Pall = np.concatenate([objs[("P", h)] for h in range(ng)], axis=1)
        a = Pall[:, g * per:(g + 1) * per]
        dx = a[0][:, None] - Pall[0][None, :]
        dy = a[1][:, None] - Pall[1][None, :]
        dz = a[2][:, None] - Pall[2][None, :]
        r2 = dx * dx + dy * dy + dz * dz + bodies.EPS2
        mag = a[3][:, None] * Pall[3][None, :] / r2
        idx = np.arange(per)
        mag[idx, g * per + idx] = 0.0
        denom = mag.sum(axis=1)
        dF = np.sqrt(((got[:3] - w[:3]) ** 2).sum(axis=0))
        assert (dF / denom).max() <= 1e-12


@pytest.mark.parametrize("b", [256, 1024])
def test_dpotrf_store_inverses_and_trsm_inverse_blocks(gpu_engine, b):
    A0 = inputs.spd_tile(51, 0, 0, b, b, b)
    A = A0.copy()
    B0 = inputs.uniform_tile(52, 0, 0, b, b, b)
    X = B0.copy()
    def run(g):
        g.task(sf.write(A), device=sf.ops.potrf_inv)
        g.task(sf.read(A), sf.write(X), device=sf.ops.trsm_inv)
    _run(gpu_engine, run)
    want = A0.copy()
    bodies.potrf_inv(want)
    L = np.tril(A)
    assert np.linalg.norm(A0 - L @ L.T) / np.linalg.norm(A0) <= 1e-12
    # the strict upper triangle of every 64x64 diagonal block holds inv(L_jj)^T
    for j0 in range(0, b, 64):
        blk, wblk = A[j0:j0 + 64, j0:j0 + 64], want[j0:j0 + 64, j0:j0 + 64]
        iu = np.triu_indices(64, 1)
        assert np.abs(blk[iu] - wblk[iu]).max() <= 1e-12 * np.abs(wblk[iu]).max()
    Xw = B0.copy()
    bodies.trsm(np.tril(want), Xw)
    assert np.linalg.norm(X - Xw) / np.linalg.norm(Xw) <= 1e-12
    assert np.linalg.norm(X @ L.T - B0) / (np.linalg.norm(L) * np.linalg.norm(X)) <= 1e-13


@pytest.mark.parametrize("sizes", [(300, 77, 1), (513, 1024, 64)])
def test_particles_ragged_groups(gpu_engine, sizes):
    """Group sizes that are not multiples of the kernel's 512-particle blocks or
    64-source chunks (padding lanes), including a one-particle group."""
    rng = np.random.default_rng(sum(sizes))
    P = [sf.pinned_empty((4, n)) for n in sizes]
    F = [sf.pinned_zeros((4, n)) for n in sizes]
    for p in P:
        p[:3] = rng.random((3, p.shape[1]))
        p[3] = 0.5 + 0.5 * rng.random(p.shape[1])
    want = [np.zeros_like(f) for f in F]
    for i in range(len(sizes)):
        bodies.p2p_self(P[i], want[i])
        for j in range(i + 1, len(sizes)):
            bodies.p2p_pair(P[i], P[j], want[i], want[j])
    _run(gpu_engine, lambda g: alg.insert_particles(g, P, F))
    for got, w in zip(F, want):
        pot_rel = np.abs(got[3] - w[3]) / np.abs(w[3])
        assert pot_rel.max() <= 1e-10, pot_rel.max()
        scale = np.abs(w[:3]).max()
        assert np.abs(got[:3] - w[:3]).max() <= 1e-11 * scale


def test_shared_commutative_members_on_gpu(gpu_engine):
    """add_i64 members of commutative groups run concurrently on the streams
    (shared guard), interleaved with exclusive members and plain writes: the
    cells equal a serial execution."""
    import random
    rng = random.Random(11)
    n = 5
    g = sf.TaskGraph().compute_on(gpu_engine)
    cells = [sf.Cell(0) for _ in range(n)]
    want = [0] * n
    for step in range(400):
        i, j = rng.sample(range(n), 2)
        if step % 80 == 79:
            g.task(sf.write(cells[i]), sf.read(cells[j]), device=sf.ops.cell("write", 2, 1))
            want[i] = (2 * want[i] + 1 + want[j]) % 10000019
        elif rng.random() < 0.2:
            g.task(sf.commutative_write(cells[i]), device=sf.ops.cell("commute", 1, 3))
            want[i] = (want[i] + 3) % 10000019
        else:
            d = rng.randrange(1, 100)
            g.task(sf.commutative_write(cells[i]), sf.commutative_write(cells[j]), device=sf.ops.add_i64(d))
            want[i] += d
            want[j] += d
    g.flush_all(keep_device=False)
    assert g.wait_all(timeout=60)
    assert [c.value for c in cells] == want


@pytest.mark.parametrize("b", [128, 512, 1024])
def test_dpotrf_full_inverse_and_one_gemm_trsm(gpu_engine, b):
    """potrf_fullinv leaves inv(L)^T in the tile's strict upper triangle; trsm_fullinv
    (one TRI-masked DGEMM + copy back) solves X L^T = B with it."""
    A0 = inputs.spd_tile(61, 0, 0, b, b, b)
    A = A0.copy()
    B0 = inputs.uniform_tile(62, 0, 0, 300, b, b)
    X = B0.copy()

    def run(g):
        g.task(sf.write(A), device=sf.ops.potrf_fullinv)
        g.task(sf.read(A), sf.write(X), device=sf.ops.trsm_fullinv)
    _run(gpu_engine, run)
    want = A0.copy()
    bodies.potrf_fullinv(want)
    L = np.tril(A)
    assert np.linalg.norm(A0 - L @ L.T) / np.linalg.norm(A0) <= 1e-12
    iu = np.triu_indices(b, 1)
    assert np.abs(A[iu] - want[iu]).max() <= 1e-12 * np.abs(want[iu]).max()
    Xw = B0.copy()
    bodies.trsm(np.tril(want), Xw)
    assert np.linalg.norm(X - Xw) / np.linalg.norm(Xw) <= 1e-12
    assert np.linalg.norm(X @ L.T - B0) / (np.linalg.norm(L) * np.linalg.norm(X)) <= 1e-13


def test_full_inverse_rejects_unsupported_sizes(gpu_engine):
    A = inputs.spd_tile(61, 0, 0, 320, 320, 320)
    g = sf.TaskGraph().compute_on(gpu_engine)
    with pytest.raises(sf.ConfigurationError):
        g.task(sf.write(A), device=sf.ops.potrf_fullinv)


@pytest.mark.parametrize("stage_stream", [0, 1])
def test_cholesky_under_a_small_arena_evicts_and_matches_oracle(stage_stream):
    """The LRU tile cache on real HBM: a working set 2.7x the arena forces
    evictions with dirty write-backs and re-staging mid-factorization; the factor
    still matches the oracle.  stage_stream = 1: the host stagings go through the
    copy stream and must wait for the write-backs of the space they reuse."""
    n, b = 2048, 256
    objs = programs.cholesky_operands(n, b)
    want = {k: v.copy() for k, v in objs.items()}
    programs.run_on_oracle(programs.cholesky_program(n // b), want, workers=4).stop()
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 4), device_memory=(36 * b * b * 8) * 10 // 27)
    eng.set_option("stage_stream", stage_stream)
    try:
        M = alg.TiledMatrix(n, b, lower=True)
        for ij, t in M.tiles.items():
            t[...] = objs[("A",) + ij]
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_cholesky(g, M)
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=120)
        st = eng.stats(0)
        assert st["evictions"] > 0 and st["writebacks"] > 0
        L = M.to_dense(lower_only=True)
        Lw = programs.assemble_lower(want, n, b)
        assert np.abs(L - Lw).max() / np.abs(Lw).max() <= 1e-12
    finally:
        eng.stop()


@pytest.mark.parametrize("window", [0, 8 << 20])
def test_staging_on_the_copy_stream_tiled_gemm_matches_numpy(window):
    """stage_stream = 1 (bench.py's e2e leg): every host->device staging copy in one
    FIFO on the copy stream, the launch groups waiting on their copies' events --
    including groups whose later tasks read a tile an earlier task of the same
    group staged.  window > 0: a group that stages waits while 8 MiB of staging
    is in flight.  Two passes over host-resident tiles, then numpy."""
    n, b = 2048, 256
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 8), device_memory=1 << 30, group_max=16)
    eng.set_option("stage_stream", 1)
    eng.set_option("stage_window", window)
    try:
        rng = np.random.default_rng(7)
        A, B, C = (alg.TiledMatrix(n, b) for _ in range(3))
        for M in (A, B):
            for t in M.tiles.values():
                t[...] = rng.standard_normal(t.shape)
        for t in C.tiles.values():
            t[...] = 0.0
        g = sf.TaskGraph().compute_on(eng)
        for _ in range(2):
            alg.insert_gemm(g, A, B, C, skew=n // b)
            for M in (C, A, B):
                for t in M.tiles.values():
                    g.flush_to_host(t)
            assert g.wait_all(timeout=120)
        want = 2.0 * (A.to_dense() @ B.to_dense())
        got = C.to_dense()
        assert np.abs(got - want).max() / np.abs(want).max() <= 1e-12
        assert eng.stats(0)["copies_to_device"] > 0
    finally:
        eng.stop()


def test_commutative_chains_scale_linearly():
    """Exclusive commutative members parked on a busy handle are handed the handle
    one at a time on release (no re-offer of every waiter on every release): 4x
    the tasks must take far less than 16x the time."""
    import time

    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 4), device_memory=1 << 28)
    try:
        def run(n):
            g = sf.TaskGraph().compute_on(eng)
            cells = [sf.Cell(0) for _ in range(4)]
            t0 = time.perf_counter()
            for _ in range(n):
                for c in cells:
                    g.task(sf.commutative_write(c), device=sf.ops.cell("commute", 1, 1))
            for c in cells:
                g.flush_to_host(c)
            assert g.wait_all(timeout=120)
            assert [c.value for c in cells] == [n] * 4
            return time.perf_counter() - t0
        run(200)
        t1, t4 = run(1000), run(4000)
        assert t4 / t1 < 8.0, (t1, t4)
    finally:
        eng.stop()


def test_read_mode_flush_keeps_the_device_copy(gpu_engine):
    """flush_to_host(keep_device=True) (reference graph.py:258-260,
    device.py:282-326): the host buffer receives the device result, the device copy
    stays valid and clean, and a later reader on the GPU stages nothing; the default
    (write-mode) flush drops the device copy, so the next reader stages again."""
    b = 256
    T = sf.pinned_zeros((b, b))
    C = sf.pinned_zeros((b, b))
    g = sf.TaskGraph().compute_on(gpu_engine)
    g.task(sf.write(T), device=sf.ops.fill_uniform(71, 0, 0, b))
    g.flush_to_host(T, keep_device=True)
    assert g.wait_all(timeout=60)
    assert np.array_equal(T, inputs.uniform_tile(71, 0, 0, b, b, b))
    hid = g.hid_of(T)
    st = gpu_engine.block_state(hid)
    assert st["present"] and st["valid"] and not st["dirty"] and st["host_valid"]
    h2d0 = gpu_engine.stats(0)["bytes_to_device"]
    g.task(sf.read(T), sf.write(C), device=sf.ops.syrk_sub)
    assert g.wait_all(timeout=60)
    # only C was staged: T's device copy was reused
    assert gpu_engine.stats(0)["bytes_to_device"] - h2d0 == b * b * 8
    g.flush_to_host(T)  # write-mode: device copies dropped
    assert g.wait_all(timeout=60)
    assert not gpu_engine.block_state(hid)["present"] or not gpu_engine.block_state(hid)["valid"]
    h2d1 = gpu_engine.stats(0)["bytes_to_device"]
    g.task(sf.read(T), sf.write(C), device=sf.ops.syrk_sub)
    assert g.wait_all(timeout=60)
    assert gpu_engine.stats(0)["bytes_to_device"] - h2d1 == b * b * 8  # T staged again


def test_million_task_soak_on_the_gpu_has_flat_runtime_memory():
    """The CUDA backend version of the simulated-backend soak: 10^6 device tasks
    (int64 cell kernels) through one history-free graph; live tasks/slots stay
    bounded, the process RSS flat, and every cell ends at its task count."""
    import psutil

    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 8), trace=False, device_memory=1 << 28)
    proc = psutil.Process()
    try:
        g = sf.TaskGraph(history=False, trace=False).compute_on(eng)
        T = 8
        cells = [sf.Cell(0) for _ in range(T)]
        H = np.array([g.hid_of(c) for c in cells], np.uint64)
        op = sf.ops.cell("write", 1, 1)
        chunk = 20000
        rss = []
        for rep in range(50):  # 50 x 20,000 = 10^6 tasks
            hids = np.tile(H, chunk // T)
            g.submit_arrays(np.full(chunk, op.code, np.uint32), np.zeros((chunk, 4)),
                            np.tile(np.array(op.iparam, np.int64), (chunk, 1)), np.zeros(chunk, np.int32),
                            np.ones(chunk, np.uint32), hids, np.full(chunk, sf.AccessMode.WRITE.code, np.uint32))
            assert g.wait_all(timeout=120)
            live = eng.live()
            assert live["tasks"] <= 4 * T and live["slots"] <= 4 * T, live
            rss.append(proc.memory_info().rss)
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=120)
        assert eng.live()["retired"] >= 10 ** 6 - 4 * T
        assert [c.value for c in cells] == [(10 ** 6 // T)] * T
        assert rss[-1] - rss[5] < 64 << 20, (rss[5], rss[-1])
    finally:
        eng.stop()


def test_commutative_gemm_accumulation_with_guards_passed_at_launch():
    """C += A_k B_k as 48 commutative_write DGEMMs over 8 streams, mixed with a few
    exclusive writes that scale C: exclusive commutative guards pass at launch on
    one device (the next member waits on the holder's end event), so members must
    still never overlap -- overlapping read-modify-write epilogues would lose
    updates.  The sum equals the serial result up to the order of additions."""
    rng = np.random.default_rng(21)
    b = 256
    A = [rng.standard_normal((b, b)) for _ in range(6)]
    B = [rng.standard_normal((b, b)) for _ in range(6)]
    C = np.zeros((b, b))
    want = np.zeros((b, b))
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 8))
    try:
        g = sf.TaskGraph().compute_on(eng)
        for rnd in range(4):
            for k in range(12):
                g.task(sf.read(A[k % 6]), sf.read(B[k % 6]), sf.commutative_write(C), device=sf.ops.gemm_nn)
                want += A[k % 6] @ B[k % 6]
            g.task(sf.read(A[0]), sf.read(B[0]), sf.write(C), device=sf.ops.dgemm(0.0, 0.5))  # C = 0.5 C
            want *= 0.5
        g.flush_to_host(C)
        assert g.wait_all(timeout=120)
    finally:
        eng.stop()
    assert np.max(np.abs(C - want)) / np.max(np.abs(want)) < 1e-12
