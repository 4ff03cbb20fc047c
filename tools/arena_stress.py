#!/usr/bin/env python
"""Tiled Cholesky through a tiny tile cache, repeated: counts wrong factors.

    python tools/arena_stress.py REPS [full|blk|none] [STREAMS] [PRIO 0/1]

2048^2 / 256 tiles (36 lower tiles of 512 KiB) through a ~7 MB arena (13 slots):
nearly every task evicts.  Environment: MEM=<arena bytes>, PF=0/1 (prefetch),
GM=<group_max>, GPS=<groups per stream>, NDEV=<logical devices on GPU 0, 2-D
block-cyclic tiles, peer pulls>, SFX_GROUP_NO_STAGE_LIMIT=1 (disable the
staging-aware launch-group limit: the regime of the write-back race in DESIGN.md §6c).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2308_15964_b200 as sf  # noqa: E402
from paper_2308_15964_b200 import algorithms as alg  # noqa: E402
from oracle import programs  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    inv = {"full": "full", "blk": True, "none": False}[sys.argv[2] if len(sys.argv) > 2 else "full"]
    streams = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    prio = (sys.argv[4] == "1") if len(sys.argv) > 4 else True
    n, b = 2048, 256
    objs = programs.cholesky_operands(n, b)
    want = {k: v.copy() for k, v in objs.items()}
    programs.run_on_oracle(programs.cholesky_program(n // b), want, workers=4).stop()
    Lw = programs.assemble_lower(want, n, b)
    mem = int(os.environ.get("MEM", (36 * b * b * 8) * 10 // 27))
    bad = 0
    for rep in range(reps):
        ndev = int(os.environ.get("NDEV", "1"))
        eng = sf.create_engine(sf.WorkerTeam.of_devices(ndev, streams), device_memory=mem, ordinals=[0] * ndev)
        for opt, env in (("prefetch", "PF"), ("group_max", "GM"), ("groups_per_stream", "GPS")):
            if os.environ.get(env) is not None:
                eng.set_option(opt, int(os.environ[env]))
        M = alg.TiledMatrix(n, b, lower=True)
        for ij, t in M.tiles.items():
            t[...] = objs[("A",) + ij]
        g = sf.TaskGraph().compute_on(eng)
        if ndev > 1:
            alg.block_cyclic(g, M, *alg.grid_shape(ndev))
        alg.insert_cholesky(g, M, priorities=prio, inverse_blocks=inv)
        g.flush_all(keep_device=False)
        g.wait_all(timeout=120)
        st = eng.stats(0)
        err = np.abs(M.to_dense(lower_only=True) - Lw).max() / np.abs(Lw).max()
        if err > 1e-12:
            bad += 1
            print(f"rep {rep}: err={err:.1e} evictions={st['evictions']} write-backs={st['writebacks']}", flush=True)
        eng.stop()
    print(f"wrong factors: {bad} of {reps}", flush=True)


if __name__ == "__main__":
    main()
