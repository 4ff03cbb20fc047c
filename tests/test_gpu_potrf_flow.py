"""The dataflow DPOTRF (csrc/kernels/potrf_flow.cu) against numpy, in its three
output modes, across tile sizes (including non-power-of-two block counts), plus
bitwise run-to-run determinism and the round-1 cooperative kernel as a second
opinion (SFX_POTRF=coop, run in a subprocess because the switch is read once).

Tolerances: ||A - L L^T||_F / ||A||_F <= 1e-12; L within 1e-12
of numpy's L (relative to max |L|); inverse blocks: max |W L - I| <= 1e-10
(an explicit inverse, error ~ cond(L) u; the SPD generator's tiles are well
conditioned).
"""

import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2308_15964_b200 as sf
from oracle import inputs

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _factor(eng, A, op):
    g = sf.TaskGraph().compute_on(eng)
    g.task(sf.write(A), device=op)
    g.flush_all(keep_device=False)
    assert g.wait_all(timeout=120)


@pytest.mark.parametrize("b", [64, 128, 192, 320, 512, 1024, 2048])
@pytest.mark.parametrize("mode", ["plain", "blocks", "full"])
def test_potrf_modes_match_numpy(gpu_engine, b, mode):
    if mode == "full" and b not in (128, 256, 512, 1024, 2048):
        pytest.skip("full inverse: power-of-two block counts (the TRSM GEMM's contract)")
    op = {"plain": sf.ops.potrf, "blocks": sf.ops.potrf_inv, "full": sf.ops.potrf_fullinv}[mode]
    A0 = inputs.spd_tile(61, 0, 0, b, b, b)
    A = A0.copy()
    _factor(gpu_engine, A, op)
    L = np.tril(A)
    assert np.linalg.norm(A0 - L @ L.T) / np.linalg.norm(A0) <= 1e-12
    Lw = np.linalg.cholesky(A0)
    assert np.abs(L - Lw).max() / np.abs(Lw).max() <= 1e-12
    iu = np.triu_indices(b, 1)
    if mode == "plain":
        assert np.array_equal(A[iu], A0[iu])  # LAPACK 'L': upper triangle untouched
    elif mode == "blocks":
        for k in range(0, b, 64):
            Lk = L[k:k + 64, k:k + 64]
            W = np.triu(A[k:k + 64, k:k + 64], 1).T + np.diag(1.0 / np.diag(Lk))
            assert np.abs(W @ Lk - np.eye(64)).max() <= 1e-10
        # off-diagonal upper blocks untouched
        for i in range(0, b, 64):
            for j in range(i + 64, b, 64):
                assert np.array_equal(A[i:i + 64, j:j + 64], A0[i:i + 64, j:j + 64])
    else:
        W = np.triu(A, 1).T + np.diag(1.0 / np.diag(L))
        assert np.abs(W @ L - np.eye(b)).max() <= 1e-10


@pytest.mark.parametrize("b", [512, 1024])
def test_potrf_is_bitwise_deterministic(gpu_engine, b):
    A0 = inputs.spd_tile(62, 0, 0, b, b, b)
    outs = []
    for _ in range(3):
        A = A0.copy()
        _factor(gpu_engine, A, sf.ops.potrf_fullinv)
        outs.append(A)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_potrf_back_to_back_on_one_stream_reuses_clean_flags(gpu_engine):
    # many factorizations in one graph: every launch must find its flags cleared
    b = 256
    tiles = [inputs.spd_tile(63 + i, 0, 0, b, b, b) for i in range(12)]
    work = [t.copy() for t in tiles]
    g = sf.TaskGraph().compute_on(gpu_engine)
    for A in work:
        g.task(sf.write(A), device=sf.ops.potrf_fullinv)
    g.flush_all(keep_device=False)
    assert g.wait_all(timeout=120)
    for A0, A in zip(tiles, work):
        L = np.tril(A)
        assert np.linalg.norm(A0 - L @ L.T) / np.linalg.norm(A0) <= 1e-12


def test_flow_and_cooperative_kernels_agree():
    # the round-1 cooperative kernel (SFX_POTRF=coop) as a second opinion on one tile
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_2308_15964_b200 as sf\n"
        "from oracle import inputs\n"
        "A = inputs.spd_tile(64, 0, 0, 1024, 1024, 1024)\n"
        "eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 2), trace=False)\n"
        "g = sf.TaskGraph().compute_on(eng)\n"
        "g.task(sf.write(A), device=sf.ops.potrf_fullinv)\n"
        "g.flush_all(keep_device=False); g.wait_all(); eng.stop()\n"
        "np.save(sys.argv[1], A)\n" % ROOT)
    outs = {}
    for variant in ("flow", "coop"):
        path = os.path.join("/tmp", f"sfx_potrf_{variant}_{os.getpid()}.npy")
        env = dict(os.environ)
        if variant == "coop":
            env["SFX_POTRF"] = "coop"
        subprocess.run([sys.executable, "-c", code, path], check=True, env=env, timeout=300)
        outs[variant] = np.load(path)
        os.unlink(path)
    Lf, Lc = np.tril(outs["flow"]), np.tril(outs["coop"])
    assert np.abs(Lf - Lc).max() / np.abs(Lc).max() <= 1e-12
    Wf, Wc = np.triu(outs["flow"], 1), np.triu(outs["coop"], 1)
    assert np.abs(Wf - Wc).max() / np.abs(Wc).max() <= 1e-10


def test_grouped_full_inverse_trsms_match_numpy():
    # independent TRSMs of one panel launch as ONE unsplit TRI-masked DGEMM (beta = 0)
    b, m = 512, 6
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 2), trace=False, group_max=8)
    try:
        A0 = inputs.spd_tile(65, 0, 0, b, b, b)
        L = A0.copy()
        Bs0 = [inputs.uniform_tile(66 + i, 0, 0, b, b, b) for i in range(m)]
        Bs = [x.copy() for x in Bs0]
        g = sf.TaskGraph().compute_on(eng)
        g.task(sf.write(L), device=sf.ops.potrf_fullinv)
        p0 = sf.gemm_paths()
        with g.gated():  # all TRSMs ready at once: one launch group
            for B in Bs:
                g.task(sf.read(L), sf.write(B), device=sf.ops.trsm_fullinv)
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=120)
        p1 = sf.gemm_paths()
        assert p1["tri"] - p0["tri"] == 1 and p1["tasks"] - p0["tasks"] == m, (p0, p1)
        assert p1["splitk"] == p0["splitk"]
        Lw = np.tril(L)
        for B0, X in zip(Bs0, Bs):
            assert np.linalg.norm(X @ Lw.T - B0) / (np.linalg.norm(Lw) * np.linalg.norm(X)) <= 1e-13
    finally:
        eng.stop()
