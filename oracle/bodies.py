"""CPU tile bodies (numpy / scipy) -- the numeric oracle and CPU baseline.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The reference contains no
tile bodies (last row), so these restate the
standard BLAS/LAPACK definitions the GPU ops implement; the reference engine
is what runs them when golden vectors are generated
(tests/golden/make_golden.py).

  gemm_nn(A, B, C)        C += A @ B                       (tiled DGEMM configs)
  gemm_nt_sub(A, B, C)    C -= A @ B.T                      (Cholesky update)
  syrk_sub(A, C)          lower(C) -= lower(A @ A.T)        (upper untouched)
  trsm(L, B)              B = B @ inv(L).T   (right, lower, transposed, non-unit)
  potrf(A)                lower(A) = cholesky(A) (reads the lower triangle only,
                          upper untouched, LAPACK dpotrf('L') semantics)
  p2p_pair(Pi, Pj, Fi, Fj, eps2)   both directions, every ordered pair once
  p2p_self(P, F, eps2)             ordered pairs a != b within the group
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

EPS2 = 1e-9


def gemm_nn(A, B, C):
    np.add(C, A @ B, out=C)


def gemm_nt_sub(A, B, C):
    np.subtract(C, A @ B.T, out=C)


def syrk_sub(A, C):
    n = C.shape[0]
    il = np.tril_indices(n)
    C[il] -= (A @ A.T)[il]


def trsm(L, B):
    B[...] = scipy.linalg.solve_triangular(L, B.T, lower=True, check_finite=False).T


def potrf(A):
    n = A.shape[0]
    low = np.tril(A)
    sym = low + np.tril(low, -1).T
    Lf = np.linalg.cholesky(sym)
    il = np.tril_indices(n)
    A[il] = Lf[il]


def potrf_inv(A, block=64):
    """potrf + inv(L_jj)^T of each 64x64 diagonal block in its strict upper triangle."""
    potrf(A)
    n = A.shape[0]
    for j0 in range(0, n, block):
        j1 = min(n, j0 + block)
        Ljj = np.tril(A[j0:j1, j0:j1])
        inv = scipy.linalg.solve_triangular(Ljj, np.eye(j1 - j0), lower=True, check_finite=False)
        iu = np.triu_indices(j1 - j0, 1)
        blk = A[j0:j1, j0:j1]
        blk[iu] = inv.T[iu]


def trsm_inv(L, B):
    """Same result as trsm (B L^-T); the operand's upper triangle is ignored."""
    trsm(np.tril(L), B)


def potrf_fullinv(A):
    """potrf + inv(L)^T of the whole factor in the strict upper triangle
    (csrc/kernels/factor_inv.cu)."""
    potrf(A)
    n = A.shape[0]
    inv = scipy.linalg.solve_triangular(np.tril(A), np.eye(n), lower=True, check_finite=False)
    iu = np.triu_indices(n, 1)
    A[iu] = inv.T[iu]


def trsm_fullinv(L, B):
    """Same result as trsm (B L^-T); the operand's upper triangle is ignored."""
    trsm(np.tril(L), B)


def _one_side(Pt, Ps, Ft, eps2, self_pair, block=512):
    """F_t += interactions on targets Pt from sources Ps."""
    nt = Pt.shape[1]
    xs, ys, zs, qs = Ps
    for a0 in range(0, nt, block):
        a1 = min(nt, a0 + block)
        dx = Pt[0, a0:a1, None] - xs[None, :]
        dy = Pt[1, a0:a1, None] - ys[None, :]
        dz = Pt[2, a0:a1, None] - zs[None, :]
        r2 = dx * dx + dy * dy + dz * dz + eps2
        inv = 1.0 / np.sqrt(r2)
        if self_pair:
            idx = np.arange(a0, a1)
            inv[idx - a0, idx] = 0.0
        qinv = qs[None, :] * inv
        s3 = qinv * inv * inv
        qa = Pt[3, a0:a1]
        Ft[0, a0:a1] += qa * (s3 * dx).sum(axis=1)
        Ft[1, a0:a1] += qa * (s3 * dy).sum(axis=1)
        Ft[2, a0:a1] += qa * (s3 * dz).sum(axis=1)
        Ft[3, a0:a1] += qinv.sum(axis=1)


def p2p_pair(Pi, Pj, Fi, Fj, eps2=EPS2):
    _one_side(Pi, Pj, Fi, eps2, False)
    _one_side(Pj, Pi, Fj, eps2, False)


def p2p_self(P, F, eps2=EPS2):
    _one_side(P, P, F, eps2, True)


def noop(*_):
    return None


BODIES = {
    "gemm_nn": gemm_nn,
    "gemm_nt_sub": gemm_nt_sub,
    "syrk_sub": syrk_sub,
    "trsm": trsm,
    "potrf": potrf,
    "potrf_inv": potrf_inv,
    "trsm_inv": trsm_inv,
    "potrf_fullinv": potrf_fullinv,
    "trsm_fullinv": trsm_fullinv,
    "p2p_pair": p2p_pair,
    "p2p_self": p2p_self,
    "noop": noop,
}

FLOPS = {
    # algorithmic flops per tile task
    "gemm_nn": lambda b: 2 * b ** 3,
    "gemm_nt_sub": lambda b: 2 * b ** 3,
    "syrk_sub": lambda b: b ** 3,
    "trsm": lambda b: b ** 3,
    "potrf": lambda b: b ** 3 / 3,
    "trsm_inv": lambda b: b ** 3,
    "potrf_inv": lambda b: b ** 3 / 3,
    "trsm_fullinv": lambda b: b ** 3,
    "potrf_fullinv": lambda b: b ** 3 / 3,
}
