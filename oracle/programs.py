"""Tile programs: the insertion loops of the north-star workloads.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  A program is a list, in
insertion order, of ``(kind, [(mode, key), ...], priority)``.  Keys name tile
handles: ``("A", i, k)``, ``("P", g)``, ...  The same program drives

* the oracle engine (oracle.stf.Oracle + oracle.bodies) -- CPU parity / baseline,
* the GPU engine (paper_2308_15964_b200.algorithms) -- the product path,
* the static successor relation (oracle.stf.static_successor_edges).

Loop orders follow SURVEY.md §8c (the order of probe A.7):

  tiled DGEMM:   for i, j, k:  C_ij += A_ik B_kj          read, read, write
  Cholesky:      for k: POTRF(A_kk) w
                        for i>k: TRSM  r(A_kk) w(A_ik)
                        for i>k: SYRK  r(A_ik) w(A_ii); for k<j<i: GEMM r(A_ik) r(A_jk) w(A_ij)
  particles:     for g: SELF r(P_g) cw(F_g);  for i<j: PAIR r(P_i) r(P_j) cw(F_i) cw(F_j)

Priorities (used only with the priority scheduler, scheduler.py:97-126): a
task is as urgent as the column of the tile it writes (earlier columns first);
writes into the current or next panel column add 10^6, which the GPU runtime
launches on its high-priority CUDA streams.
"""

from __future__ import annotations

from .stf import COMMUTE, READ, WRITE


def gemm_program(nt: int):
    prog = []
    for i in range(nt):
        for j in range(nt):
            for k in range(nt):
                prog.append(("gemm_nn", [(READ, ("A", i, k)), (READ, ("B", k, j)), (WRITE, ("C", i, j))], 0))
    return prog


def _chol_prio(nt, kind, k, i=0, j=0):
    # same rule as paper_2308_15964_b200.algorithms.cholesky_priorities
    col = {"potrf": k, "trsm": k, "syrk_sub": i, "gemm_nt_sub": j}[kind]
    bonus = {"potrf": 3, "trsm": 2, "syrk_sub": 1, "gemm_nt_sub": 0}[kind]
    p = (nt - col) * 4 + bonus + (1 if kind == "trsm" and i == k + 1 else 0)
    return p + (1_000_000 if col <= k + 1 else 0)


def cholesky_program(nt: int):
    prog = []
    for k in range(nt):
        prog.append(("potrf", [(WRITE, ("A", k, k))], _chol_prio(nt, "potrf", k)))
        for i in range(k + 1, nt):
            prog.append(("trsm", [(READ, ("A", k, k)), (WRITE, ("A", i, k))], _chol_prio(nt, "trsm", k, i)))
        for i in range(k + 1, nt):
            prog.append(("syrk_sub", [(READ, ("A", i, k)), (WRITE, ("A", i, i))], _chol_prio(nt, "syrk_sub", k, i)))
            for j in range(k + 1, i):
                prog.append(("gemm_nt_sub", [(READ, ("A", i, k)), (READ, ("A", j, k)), (WRITE, ("A", i, j))],
                             _chol_prio(nt, "gemm_nt_sub", k, i, j)))
    return prog


def particles_program(ngroups: int):
    prog = []
    for g in range(ngroups):
        prog.append(("p2p_self", [(READ, ("P", g)), (COMMUTE, ("F", g))], 0))
    for i in range(ngroups):
        for j in range(i + 1, ngroups):
            prog.append(("p2p_pair", [(READ, ("P", i)), (READ, ("P", j)), (COMMUTE, ("F", i)), (COMMUTE, ("F", j))], 0))
    return prog


def program_accesses(prog):
    return [acc for _, acc, _ in prog]


def flops(prog, b: int) -> float:
    from .bodies import FLOPS

    return float(sum(FLOPS[kind](b) for kind, _, _ in prog if kind in FLOPS))


# -- operands ------------------------------------------------------------------

def gemm_operands(n: int, b: int, seed_a: int = 1, seed_b: int = 2, alloc=None):
    """Tiles of A, B (uniform) and C = 0 as a dict key -> array."""
    import numpy as np

    from .inputs import uniform_tile

    alloc = alloc or (lambda shape: np.empty(shape))
    nt = n // b
    objs = {}
    for i in range(nt):
        for k in range(nt):
            a = alloc((b, b))
            a[...] = uniform_tile(seed_a, i * b, k * b, b, b, n)
            objs[("A", i, k)] = a
            bb = alloc((b, b))
            bb[...] = uniform_tile(seed_b, i * b, k * b, b, b, n)
            objs[("B", i, k)] = bb
            c = alloc((b, b))
            c[...] = 0.0
            objs[("C", i, k)] = c
    return objs


def cholesky_operands(n: int, b: int, seed: int = 3, alloc=None):
    import numpy as np

    from .inputs import spd_tile

    alloc = alloc or (lambda shape: np.empty(shape))
    nt = n // b
    objs = {}
    for i in range(nt):
        for j in range(i + 1):
            a = alloc((b, b))
            a[...] = spd_tile(seed, i * b, j * b, b, b, n)
            objs[("A", i, j)] = a
    return objs


def particle_operands(ngroups: int, per_group: int, seed: int = 4, alloc=None):
    import numpy as np

    from .inputs import particles

    alloc = alloc or (lambda shape: np.empty(shape))
    objs = {}
    for g in range(ngroups):
        p = alloc((4, per_group))
        p[...] = particles(seed, g * per_group, per_group)
        objs[("P", g)] = p
        f = alloc((4, per_group))
        f[...] = 0.0
        objs[("F", g)] = f
    return objs


def run_on_oracle(prog, objs, workers: int = 1, scheduler: str = "fifo", paused: bool = False,
                  bodies=True, trace: bool = True):
    """Insert ``prog`` over ``objs`` into an oracle engine; returns the finished Oracle."""
    from .bodies import BODIES
    from .stf import Oracle

    orc = Oracle(workers=workers, scheduler=scheduler, paused=paused, trace=trace)
    for kind, acc, prio in prog:
        body = BODIES[kind] if bodies else None
        orc.task([(m, objs[key]) for m, key in acc], body=body, priority=prio, name=kind)
    if paused:
        orc.resume()
    orc.wait_all()
    return orc


def assemble_lower(objs, n, b):
    """Dense lower-triangular L from Cholesky tiles (diagonal tiles' upper part zeroed)."""
    import numpy as np

    nt = n // b
    L = np.zeros((n, n))
    for i in range(nt):
        for j in range(i + 1):
            t = objs[("A", i, j)]
            L[i * b:(i + 1) * b, j * b:(j + 1) * b] = np.tril(t) if i == j else t
    return L
