"""Tiled FP64 workloads on the STF graph: DGEMM, right-looking Cholesky, particles.

These are the north-star task graphs (BASELINE.json configs).  The reference
ships no application code, so the loop orders follow
SURVEY.md §8c; each ``insert_*`` produces exactly the task sequence of a
plain loop of ``graph.task(...)`` calls -- the ``fast`` path only packs the
same descriptors into one native submission.

  tiled DGEMM   for i, j, k: C_ij += A_ik B_kj      r(A_ik) r(B_kj) w(C_ij)
  Cholesky      for k: POTRF w(A_kk); for i>k: TRSM r(A_kk) w(A_ik);
                for i>k: SYRK r(A_ik) w(A_ii); for k<j<i: GEMM r(A_ik) r(A_jk) w(A_ij)
  particles     for g: SELF r(P_g) cw(F_g); for i<j: PAIR r(P_i) r(P_j) cw(F_i) cw(F_j)
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from . import ops
from .access import commutative_write, read, write
from .memory import pinned_empty


class TiledMatrix:
    """An n x n FP64 matrix held as separate contiguous b x b host tiles.

    ``lower=True`` stores only tiles (i, j) with i >= j (Cholesky).  Tiles are
    page-locked by default so staging copies run asynchronously at full PCIe
    rate.
    """

    def __init__(self, n: int, b: int, lower: bool = False, pinned: bool = True, sim: bool = False):
        if n % b:
            raise ValueError("n must be a multiple of the tile size")
        self.n, self.b, self.nt, self.lower = n, b, n // b, lower
        alloc = (lambda: pinned_empty((b, b), np.float64, sim=sim)) if pinned else (lambda: np.empty((b, b)))
        self.tiles = {}
        for i in range(self.nt):
            for j in range(self.nt):
                if not lower or i >= j:
                    self.tiles[(i, j)] = alloc()

    def __getitem__(self, ij):
        return self.tiles[ij]

    def fill(self, value: float = 0.0):
        for t in self.tiles.values():
            t[...] = value
        return self

    def to_dense(self, lower_only: bool = False) -> np.ndarray:
        n, b = self.n, self.b
        out = np.zeros((n, n))
        for (i, j), t in self.tiles.items():
            blk = np.tril(t) if (lower_only and i == j) else t
            out[i * b:(i + 1) * b, j * b:(j + 1) * b] = blk
        return out

    @classmethod
    def from_dense(cls, a: np.ndarray, b: int, lower: bool = False, pinned: bool = True, sim: bool = False):
        m = cls(a.shape[0], b, lower=lower, pinned=pinned, sim=sim)
        for (i, j), t in m.tiles.items():
            t[...] = a[i * b:(i + 1) * b, j * b:(j + 1) * b]
        return m


class _Batch:
    """Accumulates task descriptors and submits them in one native call."""

    def __init__(self, graph):
        self.g = graph
        self.codes, self.fp, self.ip, self.prio, self.nacc, self.hids, self.modes, self.names = ([] for _ in range(8))

    def add(self, op, accesses, priority=0, name=None):
        self.codes.append(op.code)
        self.fp.append(op.fparam)
        self.ip.append(op.iparam)
        self.prio.append(priority)
        self.nacc.append(len(accesses))
        for spec in accesses:
            self.hids.append(self.g.hid_of(spec.obj))
            self.modes.append(spec.mode.code)
        self.names.append(name)

    def submit(self):
        if not self.codes:
            return np.zeros(0, np.uint64)
        return self.g.submit_arrays(np.array(self.codes, np.uint32), np.array(self.fp, np.float64),
                                    np.array(self.ip, np.int64), np.array(self.prio, np.int32),
                                    np.array(self.nacc, np.uint32), np.array(self.hids, np.uint64),
                                    np.array(self.modes, np.uint32), names=self.names)


def _emit(graph, fast):
    if fast:
        return _Batch(graph)
    return None


def insert_gemm(graph, A: TiledMatrix, B: TiledMatrix, C: TiledMatrix, fast: bool = True,
                priorities: bool = False):
    """C += A B over tiles, loop order i, j, k.

    ``priorities``: block row i gets priority nt - i, so with the priority
    scheduler the rows of C finish one after another (a few rows in flight)
    instead of every chain advancing in lock-step -- staging of A/C rows and the
    flush of finished C tiles then overlap the remaining compute.
    """
    nt = A.nt
    batch = _emit(graph, fast)
    for i in range(nt):
        for j in range(nt):
            prio = nt - i if priorities else 0
            for k in range(nt):
                acc = (read(A[i, k]), read(B[k, j]), write(C[i, j]))
                if batch:
                    batch.add(ops.gemm_nn, acc, prio, "gemm")
                else:
                    graph.task(*acc, device=ops.gemm_nn, priority=prio, name="gemm")
    return batch.submit() if batch else None


URGENT = 1_000_000  # runtime default "urgent_priority": launched on high-priority CUDA streams


def cholesky_priorities(nt: int, kind: str, k: int, i: int = 0, j: int = 0) -> int:
    """Priority of a Cholesky tile task: how soon its OUTPUT tile's column becomes a panel.

    POTRF(k) and TRSM(i,k) write column k, SYRK(i,k) writes A_ii (column i),
    GEMM(i,j,k) writes A_ij (column j).  Earlier columns first; tasks whose output
    column is the current or next panel (<= k+1) are urgent (>= URGENT): they run on
    the high-priority CUDA streams.  The next panel's TRSM is one above its
    siblings so it launches alone, ahead of the grouped rest.
    """
    col = {"potrf": k, "trsm": k, "syrk": i, "gemm": j}[kind]
    bonus = {"potrf": 3, "trsm": 2, "syrk": 1, "gemm": 0}[kind]
    p = (nt - col) * 4 + bonus
    if kind == "trsm" and i == k + 1:
        p += 1
    if col <= k + 1:
        p += URGENT
    return p


def insert_cholesky(graph, A: TiledMatrix, fast: bool = True, priorities: bool = True,
                    inverse_blocks: bool = True):
    """In-place right-looking tiled Cholesky of the lower tiles of A (A = L L^T).

    ``inverse_blocks`` (default): POTRF also leaves the inverses of its 64x64
    diagonal blocks in the diagonal tile's upper triangle and every TRSM runs as
    DMMA GEMM sweeps on them.  The factor L (lower tiles) is the same; only the
    otherwise unused upper triangle of the diagonal tiles differs.
    """
    nt = A.nt
    potrf_op = ops.potrf_inv if inverse_blocks else ops.potrf
    trsm_op = ops.trsm_inv if inverse_blocks else ops.trsm
    P = (lambda *a: cholesky_priorities(nt, *a)) if priorities else (lambda *a: 0)
    batch = _emit(graph, fast)

    def emit(op, acc, prio, name):
        if batch:
            batch.add(op, acc, prio, name)
        else:
            graph.task(*acc, device=op, priority=prio, name=name)

    for k in range(nt):
        emit(potrf_op, (write(A[k, k]),), P("potrf", k), "potrf")
        for i in range(k + 1, nt):
            emit(trsm_op, (read(A[k, k]), write(A[i, k])), P("trsm", k, i), "trsm")
        for i in range(k + 1, nt):
            emit(ops.syrk_sub, (read(A[i, k]), write(A[i, i])), P("syrk", k, i), "syrk")
            for j in range(k + 1, i):
                emit(ops.gemm_nt_sub, (read(A[i, k]), read(A[j, k]), write(A[i, j])), P("gemm", k, i, j), "gemm")
    return batch.submit() if batch else None


def insert_particles(graph, P: list, F: list, eps2: float = 1e-9, fast: bool = True):
    """All-pairs interactions between particle groups, commutative accumulation into F."""
    ng = len(P)
    batch = _emit(graph, fast)
    self_op, pair_op = ops.p2p_self(eps2), ops.p2p_pair(eps2)
    for g in range(ng):
        acc = (read(P[g]), commutative_write(F[g]))
        if batch:
            batch.add(self_op, acc, 0, "p2p_self")
        else:
            graph.task(*acc, device=self_op, name="p2p_self")
    for i in range(ng):
        for j in range(i + 1, ng):
            acc = (read(P[i]), read(P[j]), commutative_write(F[i]), commutative_write(F[j]))
            if batch:
                batch.add(pair_op, acc, 0, "p2p_pair")
            else:
                graph.task(*acc, device=pair_op, name="p2p_pair")
    return batch.submit() if batch else None


def insert_fill_uniform(graph, M: TiledMatrix, seed: int):
    """Generate uniform[0,1) tiles on the devices (bit-identical to oracle/inputs.py)."""
    batch = _Batch(graph)
    for (i, j), t in M.tiles.items():
        batch.add(ops.fill_uniform(seed, i * M.b, j * M.b, M.n), (write(t),), 0, "fill")
    return batch.submit()


def insert_fill_spd(graph, M: TiledMatrix, seed: int):
    batch = _Batch(graph)
    for (i, j), t in M.tiles.items():
        batch.add(ops.fill_spd(seed, i * M.b, j * M.b, M.n), (write(t),), 0, "fill")
    return batch.submit()


def insert_zero(graph, M: TiledMatrix):
    batch = _Batch(graph)
    for t in M.tiles.values():
        batch.add(ops.zero(), (write(t),), 0, "zero")
    return batch.submit()


def insert_fill_particles(graph, P: list, seed: int):
    batch = _Batch(graph)
    for g, p in enumerate(P):
        batch.add(ops.fill_particles(seed, g * p.shape[1]), (write(p),), 0, "fill")
    return batch.submit()


def block_cyclic(graph, M: TiledMatrix, P: int, Q: int) -> None:
    """2-D block-cyclic ownership: tile (i, j) lives on device (i % P) * Q + (j % Q).

    The locality-aware scheduler then runs every task on the owner of the tile
    it writes (owner computes) and pulls remote operands peer-to-peer.
    """
    for (i, j), t in M.tiles.items():
        graph.place(t, (i % P) * Q + (j % Q))


def grid_shape(ndev: int):
    """P x Q device grid with P <= Q, P*Q = ndev, P as large as possible (2x4 for 8)."""
    P = 1
    for p in range(1, ndev + 1):
        if ndev % p == 0 and p * p <= ndev:
            P = p
    return P, ndev // P


def flops_gemm(n: int) -> float:
    return 2.0 * n ** 3


def flops_cholesky(n: int) -> float:
    return n ** 3 / 3.0


def interactions(n_particles: int) -> float:
    return float(n_particles) * (n_particles - 1)


FLOP_PER_INTERACTION = 20

__all__ = ["TiledMatrix", "insert_gemm", "insert_cholesky", "insert_particles", "insert_fill_uniform",
           "insert_fill_spd", "insert_zero", "insert_fill_particles", "cholesky_priorities", "flops_gemm",
           "flops_cholesky", "interactions", "FLOP_PER_INTERACTION", "N"]
