"""Pin the CPU oracle to the real reference's outputs (golden fixtures).

The fixtures were produced by running the reference seqflow itself
(tests/golden/make_golden.py).  These tests need neither the reference nor a
GPU: they check that the oracle's restatement reproduces the reference's
values, successor edges, one-worker pop order, LRU resident sets and the
numbers the reference engine computed with the oracle bodies.
"""

import json
import os

import numpy as np
import pytest

from oracle import bodies, lru, programs, stf
from oracle.stf import ATOMIC, COMMUTE, MAYBE, READ, WRITE

GOLD = os.path.join(os.path.dirname(__file__), "golden")
MOD = 10_000_019
_MODE = {"read": READ, "write": WRITE, "atomic": ATOMIC, "commute": COMMUTE, "maybe": MAYBE}


def load_random_programs():
    with open(os.path.join(GOLD, "random_programs.json")) as fh:
        return json.load(fh)


def load_tile_graphs():
    return np.load(os.path.join(GOLD, "tile_graphs.npz"))


def cell_body(mode, a, b):
    """The reference random-program bodies (tests/conftest.py:87-124) on one-element lists."""
    def body(t, *rs):
        rsum = sum(r[0] for r in rs)
        if mode == "read":
            return
        if mode in ("write", "maybe"):
            if mode == "maybe" and t[0] % 2 != 0:
                return
            t[0] = (a * t[0] + b + rsum) % MOD
        elif mode == "atomic":
            t[0] = (t[0] + (b + rsum) % MOD) % MOD
        elif mode == "commute":
            t[0] = (t[0] + b + a * rsum) % MOD
    return body


def run_program_on_oracle(prog, workers=1, paused=True):
    cells = [[i + 1] for i in range(prog["n_cells"])]
    orc = stf.Oracle(workers=workers, paused=paused)
    for mode, target, reads, a, b in prog["tasks"]:
        acc = [(_MODE[mode], cells[target])] + [(READ, cells[r]) for r in reads]
        orc.task(acc, body=cell_body(mode, a, b))
    if paused:
        orc.resume()
    orc.wait_all(timeout=30)
    orc.stop()
    return orc, [c[0] for c in cells]


def test_random_programs_match_reference():
    progs = load_random_programs()
    assert len(progs) == 120
    for p in progs:
        orc, values = run_program_on_oracle(p)
        assert values == p["values"] == p["sequential"]
        assert sorted(orc.edges()) == sorted(tuple(e) for e in p["edges"])
        assert orc.pop_order() == p["pop_order"]


@pytest.mark.parametrize("workers", [2, 4, 8])
def test_random_programs_parallel_oracle(workers):
    for p in load_random_programs()[:40]:
        _, values = run_program_on_oracle(p, workers=workers, paused=False)
        assert values == p["sequential"]


def test_static_edges_restatement():
    for p in load_random_programs():
        accesses = [[(_MODE[m], t)] + [(READ, r) for r in reads] for m, t, reads, _, _ in p["tasks"]]
        assert stf.static_successor_edges(accesses) == set(tuple(e) for e in p["edges"])


@pytest.mark.parametrize("name,prog", [
    ("gemm_nt8", programs.gemm_program(8)),
    ("cholesky_nt8", programs.cholesky_program(8)),
    ("cholesky_nt32", programs.cholesky_program(32)),
    ("cholesky_nt64", programs.cholesky_program(64)),
    ("particles_g16", programs.particles_program(16)),
])
def test_tile_graph_edges_match_reference(name, prog):
    gold = load_tile_graphs()
    want = set(map(tuple, gold[f"{name}_edges"].tolist()))
    assert int(gold[f"{name}_ntasks"][0]) == len(prog)
    assert stf.static_successor_edges(programs.program_accesses(prog)) == want


@pytest.mark.parametrize("name,prog", [
    ("gemm_nt8", programs.gemm_program(8)),
    ("cholesky_nt8", programs.cholesky_program(8)),
    ("cholesky_nt32", programs.cholesky_program(32)),
    ("particles_g16", programs.particles_program(16)),
])
def test_tile_graph_pop_order_matches_reference(name, prog):
    gold = load_tile_graphs()
    keys = {}
    for _, acc, _ in prog:
        for _, k in acc:
            keys.setdefault(k, [0])
    orc = programs.run_on_oracle(prog, keys, workers=1, paused=True, bodies=False)
    orc.stop()
    assert orc.pop_order() == gold[f"{name}_pop"].tolist()
    assert orc.edges() == set(map(tuple, gold[f"{name}_edges"].tolist()))


def test_reference_lru_model_matches_reference_arena():
    with open(os.path.join(GOLD, "lru.json")) as fh:
        cases = json.load(fh)
    assert len(cases) == 230
    for c in cases:
        ref = lru.ReferenceLRU(c["capacity"])
        arena = lru.ArenaModel(c["capacity"], align=8)
        for h, want in zip(c["seq"], c["resident"]):
            ref.access(h, c["size"])
            arena.touch(h, c["size"])
            assert sorted(ref.blocks) == want
            assert sorted(arena.blocks) == want


def test_oracle_numerics_match_reference_engine():
    gold = np.load(os.path.join(GOLD, "numerics.npz"))
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        n, b = 2048, 256
        objs = programs.gemm_operands(n, b)
        programs.run_on_oracle(programs.gemm_program(n // b), objs, workers=4).stop()
        C = np.block([[objs[("C", i, j)] for j in range(n // b)] for i in range(n // b)])
        # per-tile write chains fix the summation order: bit-identical to the reference run
        assert np.array_equal(C[::17, ::19], gold["gemm_C_sample"])
        assert np.array_equal(C.sum(axis=1), gold["gemm_C_rowsum"])
        n, b = 1024, 128
        objs = programs.cholesky_operands(n, b)
        programs.run_on_oracle(programs.cholesky_program(n // b), objs, workers=4).stop()
        L = programs.assemble_lower(objs, n, b)
        assert np.array_equal(L[np.tril_indices(n)][::7], gold["chol_L"])
        ng, per = 8, 256
        objs = programs.particle_operands(ng, per)
        programs.run_on_oracle(programs.particles_program(ng), objs, workers=4).stop()
        F = np.stack([objs[("F", g)] for g in range(ng)])
        # commutative accumulation order is free: tolerance, not bits
        assert np.allclose(F, gold["particles_F"], rtol=1e-12, atol=0)


def test_oracle_bodies_definitions():
    rng = np.random.default_rng(0)
    A = rng.random((64, 64))
    B = rng.random((64, 64))
    C = rng.random((64, 64))
    C0 = C.copy()
    bodies.gemm_nt_sub(A, B, C)
    assert np.allclose(C, C0 - A @ B.T)
    S = A @ A.T + 64 * np.eye(64)
    T = S.copy()
    bodies.potrf(T)
    L = np.tril(T)
    assert np.allclose(L @ L.T, S)
    X = B.copy()
    bodies.trsm(L, X)
    assert np.allclose(X @ L.T, B)


def test_inputs_are_tiling_independent():
    from oracle import inputs

    full = inputs.uniform_tile(1, 0, 0, 64, 64, 64)
    part = inputs.uniform_tile(1, 16, 32, 16, 16, 64)
    assert np.array_equal(full[16:32, 32:48], part)
    spd = inputs.spd_tile(3, 0, 0, 64, 64, 64)
    assert np.array_equal(spd, spd.T)
    assert np.all(np.linalg.eigvalsh(spd) > 0)
    p = inputs.particles(4, 0, 100)
    assert p.shape == (4, 100) and p[3].min() >= 0.5 and p[3].max() < 1.0
