"""Output checkers for the GPU results at the BASELINE.json sizes (numpy only).

Used by ``bench.py`` (every leg verifies its own output after the timed region
and reports the numbers in its JSON line) and by the ``-m gpu`` parity tests.
Nothing here runs on the product path and nothing imports ``oracle/``: the
checkers read the operands back from the device (flushed host tiles) and apply
the size-independent properties of SURVEY.md §8d:

  DGEMM      sampled C tiles against ``m * sum_k A_ik B_kj`` (numpy/OpenBLAS):
             per-element relative error (uniform inputs: no cancellation,
             tolerance 1e-10) and the componentwise |dC| / (|A||B|) (1e-14)
  Cholesky   randomized residual ||A x - L (L^T x)|| / (||A||_F ||x||) on seeded
             vectors, O(N^2) in tile-sized pieces (tolerance 1e-12)
  particles  sampled targets against all N sources: potential relative error
             (1e-10) and |dF_a| / sum_b |F_ab| (1e-12)
"""

from __future__ import annotations

import numpy as np

GEMM_REL_TOL = 1e-10
GEMM_COMPONENTWISE_TOL = 1e-14


def gemm_componentwise_tol(n: int, passes: float = 1.0) -> float:
    """Componentwise tolerance |dC| / (|A||B|) for C accumulated over ``passes``
    products of inner dimension ``n``: 8 x the probabilistic rounding-error scale
    sqrt(n + passes) u (Higham & Mary), never below GEMM_COMPONENTWISE_TOL.  The
    fixed 1e-14 held for a few passes; a 25-pass C2 run (K = 20) measured 1.06e-14
    at n = 16384 (the per-element relative criterion, 1e-10, passed by 4 orders)."""
    return max(GEMM_COMPONENTWISE_TOL, 8.0 * (n + passes) ** 0.5 * 2.0 ** -53)
CHOL_RESIDUAL_TOL = 1e-12
POT_REL_TOL = 1e-10
FORCE_NORM_TOL = 1e-12


def gemm_tile_errors(C, A, B, samples, mult: float = 1.0, C0=None):
    """Errors of sampled output tiles of a tiled C = C0 + mult * A B.

    ``A``, ``B``, ``C`` map (i, j) -> b x b host tile (TiledMatrix.tiles);
    ``C0`` likewise or None (zero).  Returns (max per-element relative error,
    max componentwise error |dC| / (|A| |B|)).
    """
    nt = int(round(len(A) ** 0.5))
    rel = comp = 0.0
    for i, j in samples:
        want = np.zeros_like(C[i, j])
        absprod = np.zeros_like(C[i, j])
        for k in range(nt):
            want += A[i, k] @ B[k, j]
            absprod += np.abs(A[i, k]) @ np.abs(B[k, j])
        want *= mult
        absprod *= abs(mult)
        if C0 is not None:
            want += C0[i, j]
            absprod += np.abs(C0[i, j])
        d = np.abs(C[i, j] - want)
        rel = max(rel, float((d / np.abs(want)).max()))
        comp = max(comp, float((d / absprod).max()))
    return rel, comp


def sample_tiles(nt: int, count: int, seed: int = 0):
    """``count`` distinct (i, j) tile indices, always including the two corners."""
    rng = np.random.default_rng(seed)
    out = {(0, 0), (nt - 1, nt - 1)}
    while len(out) < min(count, nt * nt):
        out.add((int(rng.integers(nt)), int(rng.integers(nt))))
    return sorted(out)


def _sym_matmul(A, X, b):
    """Y = A X for a symmetric A given by its lower tiles (diagonal tiles: lower part)."""
    Y = np.zeros_like(X)
    for (i, j), t in A.items():
        xi, xj = X[i * b:(i + 1) * b], X[j * b:(j + 1) * b]
        if i == j:
            lo = np.tril(t)
            Y[i * b:(i + 1) * b] += lo @ xi + np.tril(lo, -1).T @ xi
        else:
            Y[i * b:(i + 1) * b] += t @ xj
            Y[j * b:(j + 1) * b] += t.T @ xi
    return Y


def _sym_fro2(A):
    s = 0.0
    for (i, j), t in A.items():
        if i == j:
            lo = np.tril(t)
            s += float((lo * lo).sum()) * 2 - float((np.diag(t) ** 2).sum())
        else:
            s += 2.0 * float((t * t).sum())
    return s


def cholesky_residual(A, L, n: int, b: int, nvec: int = 4, seed: int = 12):
    """max over seeded vectors x of ||A x - L (L^T x)|| / (||A||_F ||x||).

    ``A``: lower tiles of the input (before factorization); ``L``: lower tiles of
    the factor (diagonal tiles: only their lower triangle is L).  All vectors go
    through each tile at once (one pass over the tiles per product).
    """
    rng = np.random.default_rng(seed)
    anorm = _sym_fro2(A) ** 0.5
    X = rng.standard_normal((n, nvec))
    AX = _sym_matmul(A, X, b)
    Z = np.zeros_like(X)  # L^T X
    for (i, j), t in L.items():
        lt = np.tril(t) if i == j else t
        Z[j * b:(j + 1) * b] += lt.T @ X[i * b:(i + 1) * b]
    W = np.zeros_like(X)  # L Z
    for (i, j), t in L.items():
        lt = np.tril(t) if i == j else t
        W[i * b:(i + 1) * b] += lt @ Z[j * b:(j + 1) * b]
    res = np.linalg.norm(AX - W, axis=0) / (anorm * np.linalg.norm(X, axis=0))
    return float(res.max())


def particle_errors(P, F, samples, eps2: float = 1e-9, chunk: int = 1 << 18):
    """Errors of sampled targets (group g, index a) against every source.

    ``P``/``F``: lists of 4 x n SoA blocks (x, y, z, q) / (fx, fy, fz, pot).
    Returns (max potential relative error, max |dF_a| / sum_b |F_ab|).
    """
    src = np.concatenate(P, axis=1)
    offs = np.cumsum([0] + [p.shape[1] for p in P])
    pot_err = force_err = 0.0
    for g, a in samples:
        t = P[g][:, a]
        me = offs[g] + a
        pot = 0.0
        f = np.zeros(3)
        mag = 0.0
        for c0 in range(0, src.shape[1], chunk):
            s = src[:, c0:c0 + chunk]
            dx, dy, dz = t[0] - s[0], t[1] - s[1], t[2] - s[2]
            r2 = dx * dx + dy * dy + dz * dz + eps2
            inv = 1.0 / np.sqrt(r2)
            if c0 <= me < c0 + s.shape[1]:
                inv[me - c0] = 0.0
            qinv = s[3] * inv
            s3 = qinv * inv * inv
            pot += float(qinv.sum())
            f += t[3] * np.array([(s3 * dx).sum(), (s3 * dy).sum(), (s3 * dz).sum()])
            mag += float((t[3] * s3 * np.sqrt(r2 - eps2)).sum())
        got = F[g][:, a]
        pot_err = max(pot_err, abs(got[3] - pot) / abs(pot))
        force_err = max(force_err, float(np.linalg.norm(got[:3] - f)) / mag)
    return pot_err, force_err


def sample_particles(ngroups: int, per: int, count: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    out = {(0, 0), (ngroups - 1, per - 1)}
    while len(out) < count:
        out.add((int(rng.integers(ngroups)), int(rng.integers(per))))
    return sorted(out)
