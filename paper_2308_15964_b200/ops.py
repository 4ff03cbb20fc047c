"""Registered device ops: what a ``device=`` argument names in the GPU engine.

In the reference a device task is a Python callable run on a simulated-device
worker thread with ``DeviceView`` arguments (src/engine.py:144-149).  On the
B200 path a device task names one of these ops instead; its operands are the
task's declared accesses in declaration order, exactly as the reference passes
views in declaration order (README.md:50-53).  Each op is a hand-written
sm_100a kernel sequence inside libsfx.so.

Operand conventions (tiles are 2-D row-major float64 arrays):

  dgemm(alpha, beta, trans_b)   A(r), B(r), C(w):  C = beta*C + alpha*A*op(B)
  gemm_nn                       C += A @ B            (tiled DGEMM configs)
  gemm_nt_sub                   C -= A @ B.T          (Cholesky trailing update)
  dsyrk(alpha, beta)            A(r), C(w): lower(C) = beta*C + alpha*A*A^T
  syrk_sub                      lower(C) -= A @ A.T
  dtrsm()                       L(r), B(w): B = B * L^-T  (right, lower, trans)
  dpotrf()                      A(w): lower(A) = chol(A) (upper untouched, LAPACK 'L')
  dpotrf(store_inverses=True)   + inv(L_jj)^T of each 64x64 diagonal block in its strict upper
  dtrsm(inverse_blocks=True)    B = B * L^-T using those blocks (DMMA GEMM sweeps)
  p2p_pair(eps2)                P_i(r), P_j(r), F_i(cw), F_j(cw)
  p2p_self(eps2)                P_i(r), F_i(cw)
  fill_uniform/fill_spd/fill_particles/zero   generators (write one tile)
  noop, spin(ns), cell(kind, a, b), bytes_add(off, length, delta)   runtime tests
"""

from __future__ import annotations

from . import _native as N


class Op:
    """An op code plus its scalar parameters (immutable)."""

    __slots__ = ("name", "code", "fparam", "iparam")

    def __init__(self, name, code, fparam=(0.0, 0.0, 0.0, 0.0), iparam=(0, 0, 0, 0)):
        self.name = name
        self.code = code
        self.fparam = tuple(float(x) for x in (list(fparam) + [0.0] * 4)[:4])
        self.iparam = tuple(int(x) for x in (list(iparam) + [0] * 4)[:4])

    def __repr__(self):
        return f"<op {self.name}>"

    def __eq__(self, other):
        return (isinstance(other, Op) and self.code == other.code and self.fparam == other.fparam
                and self.iparam == other.iparam)

    def __hash__(self):
        return hash((self.code, self.fparam, self.iparam))


def dgemm(alpha: float = 1.0, beta: float = 1.0, trans_b: bool = False) -> Op:
    return Op("dgemm", N.OP_DGEMM, (alpha, beta), (1 if trans_b else 0,))


def dsyrk(alpha: float = -1.0, beta: float = 1.0) -> Op:
    return Op("dsyrk", N.OP_DSYRK, (alpha, beta))


def dtrsm(inverse_blocks=False) -> Op:
    """B = B L^-T.  ``inverse_blocks=True``: L's tile comes from ``dpotrf(store_inverses=True)``
    and carries the inverses of its 64x64 diagonal blocks in its upper triangle, so the
    solve runs as DMMA GEMM sweeps (x inverse block, then trailing update).
    ``inverse_blocks="full"``: L's tile comes from ``dpotrf(store_inverses="full")`` and
    carries inv(L)^T in its strict upper triangle: the solve is ONE parallel DMMA GEMM."""
    if inverse_blocks == "full":
        return Op("dtrsm_fullinv", N.OP_DTRSM, iparam=(2,))
    return Op("dtrsm_inv" if inverse_blocks else "dtrsm", N.OP_DTRSM, iparam=(1 if inverse_blocks else 0,))


def dpotrf(store_inverses=False) -> Op:
    """Lower Cholesky in place.  Default: LAPACK 'L' semantics (upper triangle untouched).
    ``store_inverses=True``: the strict upper triangle of each 64x64 diagonal block receives
    inv(L_jj)^T (for ``dtrsm(inverse_blocks=True)``); ``"full"``: the whole strict upper
    triangle receives inv(L)^T (n = 64 * 2^k, 128 <= n <= 2048; for
    ``dtrsm(inverse_blocks="full")``).  The factor L is identical in every mode."""
    if store_inverses == "full":
        return Op("dpotrf_fullinv", N.OP_DPOTRF, iparam=(2,))
    return Op("dpotrf_inv" if store_inverses else "dpotrf", N.OP_DPOTRF, iparam=(1 if store_inverses else 0,))


def p2p_pair(eps2: float = 1e-9) -> Op:
    return Op("p2p_pair", N.OP_P2P_PAIR, (eps2,))


def p2p_self(eps2: float = 1e-9) -> Op:
    return Op("p2p_self", N.OP_P2P_SELF, (eps2,))


def fill_uniform(seed: int, row0: int, col0: int, ncols_total: int) -> Op:
    return Op("fill_uniform", N.OP_FILL_UNIFORM, iparam=(seed, row0, col0, ncols_total))


def fill_spd(seed: int, row0: int, col0: int, n: int) -> Op:
    return Op("fill_spd", N.OP_FILL_SPD, iparam=(seed, row0, col0, n))


def fill_particles(seed: int, first: int) -> Op:
    return Op("fill_particles", N.OP_FILL_PARTICLES, iparam=(seed, first))


def zero() -> Op:
    return Op("zero", N.OP_ZERO)


def dacc() -> Op:
    """A += B1 + ... + Bk (k <= 7): sums per-GPU partial accumulators into their target."""
    return Op("dacc", N.OP_DACC)


def spin(ns: int) -> Op:
    return Op("spin", N.OP_SPIN, iparam=(int(ns),))


def cell(kind: str, a: int = 1, b: int = 0) -> Op:
    """Cell arithmetic of the reference random programs (tests/conftest.py:87-124)."""
    kinds = {"read": 0, "write": 1, "maybe": 2, "atomic": 3, "commute": 4}
    return Op(f"cell_{kind}", N.OP_CELL, iparam=(kinds[kind], a, b))


def bytes_add(off: int, length: int, delta: int) -> Op:
    return Op("bytes_add", N.OP_BYTES_ADD, iparam=(off, length, delta))


def add_i64(delta: int) -> Op:
    """Every operand (an int64 cell) += delta with device atomics.  An op that
    accumulates atomically: its commutative_write members of one group run
    concurrently on one device (shared guard; the P2P ops behave the same)."""
    return Op("add_i64", N.OP_ADD_I64, iparam=(int(delta),))


def fault(kind: str = "launch") -> Op:
    """Failure injection (engine-failure tests): ``"launch"`` = a kernel launch with an
    invalid configuration (the launch fails; the CUDA context survives), ``"trap"`` = a
    device-side trap (sticky: the process's CUDA context is lost)."""
    return Op(f"fault_{kind}", N.OP_FAULT, iparam=({"launch": 0, "trap": 1}[kind],))


noop = Op("noop", N.OP_NOOP)
gemm_nn = dgemm(1.0, 1.0, False)
gemm_nt_sub = dgemm(-1.0, 1.0, True)
syrk_sub = dsyrk(-1.0, 1.0)
trsm = dtrsm()
potrf = dpotrf()
trsm_inv = dtrsm(inverse_blocks=True)
potrf_inv = dpotrf(store_inverses=True)
trsm_fullinv = dtrsm(inverse_blocks="full")
potrf_fullinv = dpotrf(store_inverses="full")
