"""The vectorised insertion paths (algorithms.insert_*(fast=True)) submit exactly
the task sequence of the plain per-task loops (graph.task), chunk by chunk.

Both paths are intercepted just before the native submit, so this runs on CPU
with any op (the simulated backend would reject DGEMM/P2P at submit time).
"""

import numpy as np
import pytest

import paper_2308_15964_b200 as sf
from paper_2308_15964_b200 import algorithms as alg


def _capture(graph):
    seq = []

    def submit_arrays(codes, fp, ip, prio, nacc, hids, modes, devices=None, names=None):
        k = 0
        for t in range(len(codes)):
            n = int(nacc[t])
            seq.append((int(codes[t]), tuple(np.asarray(fp[t]).tolist()), tuple(np.asarray(ip[t]).tolist()),
                        int(prio[t]), tuple(int(h) for h in hids[k:k + n]), tuple(int(m) for m in modes[k:k + n])))
            k += n
        return np.arange(len(codes), dtype=np.uint64)

    def submit_one(tid, op, priority, hids, modes, dev_hint=-1):
        seq.append((op.code, op.fparam, op.iparam, int(priority),
                    tuple(hids), tuple(modes)))

    graph.submit_arrays = submit_arrays
    graph._submit_one = submit_one
    graph._hval = None  # no native task() fast path: every task goes through _submit_one
    return seq


@pytest.fixture
def engine():
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 2), backend="sim")
    yield eng
    eng.stop()


def _norm(seq):
    return [(c, tuple(float(x) for x in fp), tuple(int(x) for x in ip), p, h, m) for c, fp, ip, p, h, m in seq]


@pytest.mark.parametrize("priorities", [False, True])
def test_gemm_fast_matches_loop(engine, priorities):
    A, B, C = (alg.TiledMatrix(64, 16, pinned=False, sim=True) for _ in range(3))
    g = sf.TaskGraph().compute_on(engine)
    seq = _capture(g)
    alg.insert_gemm(g, A, B, C, fast=False, priorities=priorities)
    slow = _norm(seq)
    seq.clear()
    alg.insert_gemm(g, A, B, C, fast=True, priorities=priorities)
    assert _norm(seq) == slow
    assert len(slow) == 4 ** 3


@pytest.mark.parametrize("skew,skew_block", [(4, 0), (12, 2), (12, 3)])
def test_gemm_skew_priorities_fast_matches_loop(engine, skew, skew_block):
    # wavefront priorities (bench.py's e2e leg): task (i, j, k) gets -(k + offset of
    # chain (i, j)); with skew_block h the chains are ranked in h x h blocks
    nt = 4
    A, B, C = (alg.TiledMatrix(nt * 16, 16, pinned=False, sim=True) for _ in range(3))
    g = sf.TaskGraph().compute_on(engine)
    seq = _capture(g)
    alg.insert_gemm(g, A, B, C, fast=False, skew=skew, skew_block=skew_block)
    slow = _norm(seq)
    seq.clear()
    alg.insert_gemm(g, A, B, C, fast=True, skew=skew, skew_block=skew_block)
    assert _norm(seq) == slow
    # loop order i, j, k: the chain offsets, in block order when skew_block > 0
    offs = {}
    for n, (_, _, _, p, _, _) in enumerate(slow):
        i, j, k = n // (nt * nt), (n // nt) % nt, n % nt
        offs.setdefault((i, j), -p - k)
        assert -p - k == offs[(i, j)]
    h = skew_block or nt
    order = sorted(offs, key=lambda ij: (ij[0] // h, ij[1] // h, ij[0], ij[1]) if skew_block else ij)
    assert [offs[c] for c in order] == [skew * r // (nt * nt) for r in range(nt * nt)]


def test_cholesky_fast_matches_loop(engine):
    A = alg.TiledMatrix(80, 16, lower=True, pinned=False, sim=True)
    g = sf.TaskGraph().compute_on(engine)
    seq = _capture(g)
    alg.insert_cholesky(g, A, fast=False)
    slow = _norm(seq)
    seq.clear()
    alg.insert_cholesky(g, A, fast=True)
    assert _norm(seq) == slow
    nt = 5
    assert len(slow) == nt + nt * (nt - 1) // 2 * 2 + sum((i - 1) * i // 2 for i in range(nt))


def test_particles_fast_matches_loop(engine):
    P = [np.zeros((4, 8)) for _ in range(7)]
    F = [np.zeros((4, 8)) for _ in range(7)]
    g = sf.TaskGraph().compute_on(engine)
    seq = _capture(g)
    alg.insert_particles(g, P, F, fast=False)
    slow = _norm(seq)
    seq.clear()
    alg.insert_particles(g, P, F, fast=True)
    assert _norm(seq) == slow
    assert len(slow) == 7 + 21


def test_chunked_submission_names_and_ids(engine):
    """Array submissions keep one name per block and report every task id."""
    g = sf.TaskGraph().compute_on(engine)
    cells = [np.zeros(1, np.int64) for _ in range(3)]
    from paper_2308_15964_b200 import ops
    from paper_2308_15964_b200.access import AccessMode
    batch = alg._Batch(g)
    hids = np.array([[g.hid_of(c)] for c in cells], np.uint64)
    batch.add_many(ops.noop, hids, (AccessMode.WRITE.code,), 0, "blk")
    batch.flush()
    batch.add(ops.noop, (sf.read(cells[0]),), 0, "single")
    tids = batch.submit()
    assert len(tids) == 4
    assert g.wait_all(timeout=30)
    assert [g._label(int(t)) for t in tids] == ["blk", "blk", "blk", "single"]
    assert sorted(int(t) for t in tids) == [t for t in g.all_task_ids() if t in set(int(x) for x in tids)]
