"""Deterministic mode ("the reduction order is fixed in
deterministic mode, so repeated GPU runs are bitwise identical"): one GPU, one
stream, FIFO, ``create_engine(deterministic=True)`` -- particle ops run the
one-sided atomic-free kernel under exclusive commutative guards, DGEMMs never
split K.  Repeated runs must agree bit for bit and still match the oracle within
the stated tolerances (-m gpu)."""

import numpy as np
import pytest

import paper_2308_15964_b200 as sf
from paper_2308_15964_b200 import algorithms as alg
from oracle import inputs, programs

pytestmark = pytest.mark.gpu


def _det_engine():
    return sf.create_engine(sf.WorkerTeam.of_devices(1, 1), scheduler=None, device_memory=2 << 30,
                            deterministic=True)


def _particles(det: bool, ng=6, per=700):
    objs = programs.particle_operands(ng, per)
    eng = _det_engine() if det else sf.create_engine(sf.WorkerTeam.of_devices(1, 8), device_memory=2 << 30)
    try:
        P = [sf.pinned_empty((4, per)) for _ in range(ng)]
        F = [sf.pinned_zeros((4, per)) for _ in range(ng)]
        for g in range(ng):
            P[g][...] = objs[("P", g)]
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_particles(g, P, F)
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=120)
    finally:
        eng.stop()
    return objs, np.stack(F)


def test_particles_deterministic_bitwise_and_within_tolerance():
    objs, F1 = _particles(True)
    _, F2 = _particles(True)
    assert np.array_equal(F1, F2)  # bitwise identical
    ng, per = F1.shape[0], F1.shape[2]
    want = {k: v.copy() for k, v in objs.items()}
    programs.run_on_oracle(programs.particles_program(ng), want, workers=2).stop()
    for g in range(ng):
        w = want[("F", g)]
        assert (np.abs(F1[g][3] - w[3]) / np.abs(w[3])).max() <= 1e-10
        assert np.abs(F1[g][:3] - w[:3]).max() <= 1e-11 * np.abs(w[:3]).max()


def _cholesky(b=1024, n=2048):
    eng = _det_engine()
    try:
        M = alg.TiledMatrix(n, b, lower=True)
        g = sf.TaskGraph().compute_on(eng)
        alg.insert_fill_spd(g, M, 3)
        alg.insert_cholesky(g, M)
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=120)
        return M.to_dense()
    finally:
        eng.stop()


def test_cholesky_and_split_k_gemm_deterministic_bitwise():
    """b = 1024 Cholesky: its full-inverse TRSM (TRI split) and POTRF doubling
    GEMMs would split K with FP64 atomics; in deterministic mode they do not."""
    before = sf.gemm_paths()
    L1 = _cholesky()
    d = {k: sf.gemm_paths()[k] - before[k] for k in before}
    assert d["splitk"] == 0, d
    L2 = _cholesky()
    assert np.array_equal(L1, L2)
    n = L1.shape[0]
    A = np.zeros((n, n))
    for i in range(0, n, 1024):
        for j in range(0, i + 1, 1024):
            A[i:i + 1024, j:j + 1024] = inputs.spd_tile(3, i, j, 1024, 1024, n)
    A = np.tril(A) + np.tril(A, -1).T
    assert np.linalg.norm(A - L1 @ L1.T) / np.linalg.norm(A) <= 1e-12
