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
from .access import AccessMode, commutative_write, read, write
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

    def to_dense(self, lower_only=None) -> np.ndarray:
        """Dense copy of the host tiles.  ``lower_only`` (default: True for a lower
        matrix) keeps only the lower triangle of the diagonal tiles: after
        ``insert_cholesky`` with the default full-inverse POTRF their strict upper
        triangle holds inv(L)^T (a by-product the TRSMs read), where the reference
        program leaves the input there (LAPACK 'L' semantics for the lower part)."""
        if lower_only is None:
            lower_only = self.lower
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
    """Accumulates task descriptors and submits them in native calls.

    ``add`` takes one task (access specs); ``add_many`` takes a regular block of
    tasks as arrays (one row of handle ids per task), built with numpy so that
    the host cost per task is a few ns.  ``flush`` submits what is pending, so
    long loops can hand work to the executors chunk by chunk while the rest is
    still being built (insertion overlaps execution; program order is kept).
    """

    def __init__(self, graph):
        self.g = graph
        self._chunks = []  # (codes, fp, ip, prio, nacc, hids, modes, name-or-list)
        self._single = None
        self._tids = []

    def _single_lists(self):
        if self._single is None:
            self._single = tuple([] for _ in range(8))
        return self._single

    def add(self, op, accesses, priority=0, name=None):
        codes, fp, ip, prio, nacc, hids, modes, names = self._single_lists()
        codes.append(op.code)
        fp.append(op.fparam)
        ip.append(op.iparam)
        prio.append(priority)
        nacc.append(len(accesses))
        for spec in accesses:
            hids.append(self.g.hid_of(spec.obj))
            modes.append(spec.mode.code)
        names.append(name)

    def _close_single(self):
        if self._single is not None and self._single[0]:
            codes, fp, ip, prio, nacc, hids, modes, names = self._single
            self._chunks.append((np.array(codes, np.uint32), np.array(fp, np.float64), np.array(ip, np.int64),
                                 np.array(prio, np.int32), np.array(nacc, np.uint32), np.array(hids, np.uint64),
                                 np.array(modes, np.uint32), names))
        self._single = None

    def add_many(self, op, hids, modes, priority=0, name=None):
        """``hids``: (n, k) handle ids, row t = task t's accesses in declaration
        order; ``modes``: the k access mode codes; ``priority``: scalar or (n,)."""
        self._close_single()
        hids = np.ascontiguousarray(hids, dtype=np.uint64)
        n, k = hids.shape
        if n == 0:
            return
        self._chunks.append((np.full(n, op.code, np.uint32), np.broadcast_to(np.array(op.fparam), (n, 4)),
                             np.broadcast_to(np.array(op.iparam, np.int64), (n, 4)),
                             np.broadcast_to(np.asarray(priority, np.int32), (n,)), np.full(n, k, np.uint32),
                             hids.reshape(-1), np.tile(np.asarray(modes, np.uint32), n), name))

    def flush(self):
        self._close_single()
        if not self._chunks:
            return
        ch, self._chunks = self._chunks, []
        cat = [np.concatenate([c[f] for c in ch]) for f in range(7)]
        names = ch[0][7] if len(ch) == 1 else None  # a block name (str) or per-task list
        if len(ch) > 1 and any(c[7] is not None for c in ch):
            names = []
            for c in ch:
                names.extend(c[7] if isinstance(c[7], list) else [c[7]] * len(c[0]))
        self._tids.append(self.g.submit_arrays(*cat, names=names))

    def submit(self):
        self.flush()
        if not self._tids:
            return np.zeros(0, np.uint64)
        return np.concatenate(self._tids)


def _hid_grid(graph, M):
    """Handle ids of M's tiles as an (nt, nt) array (0 where a lower matrix has no tile)."""
    H = np.zeros((M.nt, M.nt), np.uint64)
    for (i, j), t in M.tiles.items():
        H[i, j] = graph.hid_of(t)
    return H


def _emit(graph, fast):
    if fast:
        return _Batch(graph)
    return None


def insert_gemm(graph, A: TiledMatrix, B: TiledMatrix, C: TiledMatrix, fast: bool = True,
                priorities=False, tile_block: int = 0, skew: int = 0, skew_block: int = 0,
                prio_base: int = 0):
    """C += A B over tiles, loop order i, j, k.

    ``priorities`` (False, True or a row-block height h): block row i gets priority
    (nt - i) // h (h = 1 for True), so with the priority
    scheduler the rows of C finish one after another (a few rows in flight)
    instead of every chain advancing in lock-step -- staging of A/C rows and the
    flush of finished C tiles then overlap the remaining compute.

    ``skew`` = S > 0 (overrides the others): a wavefront -- task (i, j, k) gets
    priority -(k + S * (i * nt + j) // nt^2), so the k-chains of the C tiles start
    staggered over S waves: when the operands start on the host, C's staging and
    its final flush spread over the run instead of piling up in the first and
    last waves.

    ``skew_block`` = h > 0 (with ``skew``): the chains take their offsets in h x h
    block order (block-row-major, row-major inside a block) instead of row-major
    order, so the first waves' chains share h rows of A and h columns of B.

    ``tile_block`` = h > 0 (overrides ``priorities``): the C tiles are ranked in
    h x h blocks (block-row-major), each block's tasks one priority level above the
    next block's: a block needs only h rows of A and h columns of B, so when the
    operands start on the host, staging spreads over the whole step.

    ``prio_base`` is added to every task's priority (a stream of products
    inserted back to back: each later product strictly below the earlier ones).
    """
    nt = A.nt
    if skew:
        if skew_block:
            hb = int(skew_block)

            def chain_rank(i, j):
                bi, bj = i // hb, j // hb
                bh = min(hb, nt - bi * hb)  # rows in this block row
                bw = min(hb, nt - bj * hb)
                return bi * hb * nt + bj * hb * bh + (i - bi * hb) * bw + (j - bj * hb)
            off = lambda i, j: int(skew) * chain_rank(i, j) // (nt * nt)  # noqa: E731
        else:
            off = lambda i, j: int(skew) * (i * nt + j) // (nt * nt)  # noqa: E731
    if tile_block:
        h = int(tile_block)
        nbc = (nt + h - 1) // h
        nblocks = nbc * nbc
        rank = lambda i, j: nblocks - ((i // h) * nbc + j // h)  # noqa: E731
    elif priorities:
        rank = lambda i, j: (nt - i) // int(priorities)  # noqa: E731
    else:
        rank = lambda i, j: 0  # noqa: E731
    if not fast:
        for i in range(nt):
            for j in range(nt):
                for k in range(nt):
                    prio = (-(k + off(i, j)) if skew else rank(i, j)) + prio_base
                    graph.task(read(A[i, k]), read(B[k, j]), write(C[i, j]), device=ops.gemm_nn,
                               priority=prio, name="gemm")
        return None
    # same (i, j, k) task sequence, built as arrays and submitted one block row
    # of C at a time so the executors start while later rows are being built
    HA, HB, HC = _hid_grid(graph, A), _hid_grid(graph, B), _hid_grid(graph, C)
    modes = (AccessMode.READ.code, AccessMode.READ.code, AccessMode.WRITE.code)
    batch = _Batch(graph)
    jj, kk = np.meshgrid(np.arange(nt), np.arange(nt), indexing="ij")
    jj, kk = jj.reshape(-1), kk.reshape(-1)
    for i in range(nt):
        hids = np.stack([HA[i, kk], HB[kk, jj], HC[i, jj]], axis=1)
        if skew:  # per task: -(k + offset of its chain)
            prio = -(kk + np.array([off(i, j) for j in range(nt)], np.int64)[jj]).astype(np.int32)
        else:
            prio = np.repeat(np.array([rank(i, j) for j in range(nt)], np.int32), nt)  # jj-major like hids
        if prio_base:
            prio = prio + np.int32(prio_base)
        batch.add_many(ops.gemm_nn, hids, modes, prio, "gemm")
        batch.flush()
    return batch.submit()


URGENT = 1_000_000  # runtime default "urgent_priority": launched on high-priority CUDA streams


def cholesky_priorities_critical(nt: int, kind: str, k: int, i: int = 0, j: int = 0) -> int:
    """Critical-path-only priorities: the tasks writing the current or next panel
    column (POTRF(k), TRSM(., k), updates of column k+1) are urgent (high-priority
    streams, popped first); every other task keeps priority 0, i.e. FIFO
    order of readiness, which keeps the ready queue's same-shape runs long
    (bigger grouped launches)."""
    col = {"potrf": k, "trsm": k, "syrk": i, "gemm": j}[kind]
    if col > k + 1:
        return 0
    bonus = {"potrf": 3, "trsm": 2, "syrk": 1, "gemm": 0}[kind]
    p = URGENT + (nt - col) * 4 + bonus
    if kind == "trsm" and i == k + 1:
        p += 1
    return p


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


def fullinv_tile(b: int) -> bool:
    """Tile sizes the full-inverse POTRF/TRSM pair supports (64 * 2^k, 128..2048)."""
    nb = b // 64
    return b % 64 == 0 and 128 <= b <= 2048 and nb & (nb - 1) == 0


def insert_cholesky(graph, A: TiledMatrix, fast: bool = True, priorities="auto",
                    inverse_blocks="auto"):
    """In-place right-looking tiled Cholesky of the lower tiles of A (A = L L^T).

    The diagonal tiles' strict upper triangle: with the default full-inverse POTRF
    it receives inv(L)^T (a by-product the TRSMs read); ``inverse_blocks=False``
    leaves it untouched like the reference's LAPACK-'L' program.  The factor L
    (the lower tiles and the diagonal tiles' lower triangle) is the same in every
    mode; ``TiledMatrix.to_dense()`` returns only L for lower matrices.

    ``inverse_blocks``: True = POTRF also leaves the inverses of its 64x64
    diagonal blocks in the diagonal tile's upper triangle and every TRSM runs as
    DMMA GEMM sweeps on them; "full" = POTRF leaves inv(L)^T of the whole tile
    there and every TRSM is one parallel DMMA GEMM (the panel chain's latency:
    TRSM 1024 770 -> ~100 us); "auto" (default) = "full" where the tile size
    allows it, else True; False = plain substitution kernels.  The factor L
    (lower tiles) is the same; only the otherwise unused upper triangle of the
    diagonal tiles differs.

    ``priorities``: True = column priorities (cholesky_priorities), "critical" =
    critical-path tasks only, False = all 0 (FIFO readiness order), "auto" = False
    on one GPU, True on several.  Priorities never change the task graph: the
    dependency edges and the factor are identical.
    """
    nt = A.nt
    if priorities == "auto":
        # measured on one B200 (tools/chol_sweep.py): when the matrix fits in the tile
        # cache, FIFO readiness order beats the column priorities (C3 30.8 vs 28.8,
        # C5 33.4 vs 31.1 TFLOP/s): long runs of same-shape ready tasks make big
        # grouped launches and the streams stay full.  When it does not fit, the
        # column order keeps the LRU working set small (C3 with a 3 GiB arena for its
        # 4.1 GiB of tiles: 25.9 vs 17.1 TFLOP/s, 4x fewer dirty write-backs).  Across
        # GPUs the column priorities keep the panel chain ahead of the owner-computes
        # updates (untested on hardware: single-GPU boxes only).
        eng = getattr(graph, "engine", None)
        ndev = getattr(eng, "ndev", 1) if eng is not None else 1
        priorities = ndev > 1
        if not priorities and eng is not None and getattr(eng, "backend", "cuda") == "cuda":
            need = sum(t.nbytes for t in A.tiles.values())
            cap = sum(eng.stats(d)["capacity"] for d in range(ndev))
            priorities = need > 0.8 * cap
    if inverse_blocks == "auto":
        inverse_blocks = "full" if fullinv_tile(A.b) else True
    if inverse_blocks == "full":
        potrf_op, trsm_op = ops.potrf_fullinv, ops.trsm_fullinv
    else:
        potrf_op = ops.potrf_inv if inverse_blocks else ops.potrf
        trsm_op = ops.trsm_inv if inverse_blocks else ops.trsm
    if priorities == "critical":
        P = lambda *a: cholesky_priorities_critical(nt, *a)  # noqa: E731
    elif priorities:
        P = lambda *a: cholesky_priorities(nt, *a)  # noqa: E731
    else:
        P = lambda *a: 0  # noqa: E731
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
        if batch:
            batch.flush()  # hand step k to the executors while step k+1 is built
    return batch.submit() if batch else None


def insert_particles(graph, P: list, F: list, eps2: float = 1e-9, fast: bool = True, devices=None,
                     partials=None):
    """All-pairs interactions between particle groups, commutative accumulation into F.

    On one GPU every task accumulates into F directly (commutative groups, shared
    guards: the kernel's updates are device atomics).  With ``devices`` > 1 (default:
    the engine's device count) the program follows SURVEY.md §8e: device d > 0 gets
    private zeroed partial accumulators Fd[g] (homed on d), the pair tasks are dealt
    to the devices in balanced contiguous blocks (positions replicate lazily by
    peer pulls, 128 KiB per group), device 0 accumulates into F itself, and one
    ``dacc`` task per group adds the partials into F[g] (peer pulls of 128 KiB per
    partial).  Returns the list of partial accumulators (keep them alive until
    wait_all) or None.
    """
    ng = len(P)
    self_op, pair_op = ops.p2p_self(eps2), ops.p2p_pair(eps2)
    if devices is None:
        eng = getattr(graph, "engine", None)
        devices = getattr(eng, "ndev", 1) if eng is not None else 1
    if devices > 1:
        return _insert_particles_multi(graph, P, F, self_op, pair_op, min(devices, 8), partials)
    if not fast:
        for g in range(ng):
            graph.task(read(P[g]), commutative_write(F[g]), device=self_op, name="p2p_self")
        for i in range(ng):
            for j in range(i + 1, ng):
                graph.task(read(P[i]), read(P[j]), commutative_write(F[i]), commutative_write(F[j]),
                           device=pair_op, name="p2p_pair")
        return None
    HP = np.array([graph.hid_of(p) for p in P], np.uint64)
    HF = np.array([graph.hid_of(f) for f in F], np.uint64)
    R, CW = AccessMode.READ.code, AccessMode.COMMUTATIVE_WRITE.code
    batch = _Batch(graph)
    batch.add_many(self_op, np.stack([HP, HF], axis=1), (R, CW), 0, "p2p_self")
    batch.flush()
    ii, jj = np.triu_indices(ng, 1)  # (i, j) pairs in loop order
    pairs = np.stack([HP[ii], HP[jj], HF[ii], HF[jj]], axis=1)
    for c0 in range(0, len(pairs), 4096):  # chunks: execution starts while the rest is submitted
        batch.add_many(pair_op, pairs[c0:c0 + 4096], (R, R, CW, CW), 0, "p2p_pair")
        batch.flush()
    return batch.submit()


def _insert_particles_multi(graph, P, F, self_op, pair_op, ndev, partials=None):
    ng = len(P)
    for f in F:
        graph.place(f, 0)
    if partials is None or len(partials) != ndev - 1:
        partials = [[pinned_empty(f.shape, np.float64) for f in F] for _ in range(1, ndev)]
    for d, Fd in enumerate(partials, start=1):
        for f in Fd:
            graph.place(f, d)
            graph.task(write(f), device=ops.zero(), name="zero_partial")
    acc = [F] + partials  # acc[d][g]: device d's accumulator of group g

    HP = np.array([graph.hid_of(p) for p in P], np.uint64)
    HF = np.array([[graph.hid_of(f) for f in acc[d]] for d in range(ndev)], np.uint64)
    R, CW = AccessMode.READ.code, AccessMode.COMMUTATIVE_WRITE.code
    batch = _Batch(graph)
    # self tasks round-robin, pair tasks in contiguous balanced blocks (consecutive
    # tasks on a device then reuse each other's source groups)
    gg = np.arange(ng)
    batch.add_many(self_op, np.stack([HP, HF[gg % ndev, gg]], axis=1), (R, CW), 0, "p2p_self")
    batch.flush()
    ii, jj = np.triu_indices(ng, 1)
    dd = np.arange(len(ii)) * ndev // len(ii)
    pairs = np.stack([HP[ii], HP[jj], HF[dd, ii], HF[dd, jj]], axis=1)
    for c0 in range(0, len(pairs), 4096):
        batch.add_many(pair_op, pairs[c0:c0 + 4096], (R, R, CW, CW), 0, "p2p_pair")
        batch.flush()
    batch.submit()
    for g in range(ng):
        graph.task(write(F[g]), *[read(acc[d][g]) for d in range(1, ndev)], device=ops.dacc(), name="reduce")
    return partials


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
