"""Tiled Cholesky on N (logical) devices from one runtime, checked by the randomized
residual (verify.py); knobs from the environment.  A debugging / stress tool:

    ORD=0,0 N=32768 B=1024 STREAMS=32 GROUP=8 REPS=3 python tools/chol_multi_check.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2308_15964_b200 as sf  # noqa: E402
import verify  # noqa: E402
from paper_2308_15964_b200 import algorithms as alg  # noqa: E402

ords = [int(x) for x in os.environ.get("ORD", "0,0").split(",")]
n, b = int(os.environ.get("N", 32768)), int(os.environ.get("B", 1024))
streams, group = int(os.environ.get("STREAMS", 32)), int(os.environ.get("GROUP", 8))
reps = int(os.environ.get("REPS", 3))
prio = os.environ.get("PRIO", "auto")
prio = {"auto": "auto", "1": True, "0": False}.get(prio, prio)
eng = sf.create_engine(sf.WorkerTeam.of_devices(len(ords), streams), scheduler="prio", trace=False,
                       ordinals=ords, group_max=group,
                       device_memory=int(os.environ["ARENA"]) if "ARENA" in os.environ else None)
for k, v in os.environ.items():
    if k.startswith("OPT_"):
        eng.set_option(k[4:].lower(), int(v))
M = alg.TiledMatrix(n, b, lower=True)
P, Q = alg.grid_shape(len(ords))
bad = 0
for rep in range(reps):
    g = sf.TaskGraph().compute_on(eng)
    if len(ords) > 1:
        alg.block_cyclic(g, M, P, Q)
    alg.insert_fill_spd(g, M, 3)
    g.flush_all(keep_device=True)
    g.wait_all()
    A = {ij: t.copy() for ij, t in M.tiles.items()}
    t0 = time.time()
    try:
        alg.insert_cholesky(g, M, priorities=prio)
        g.flush_all(keep_device=False)
        g.wait_all()
    except sf.EngineFailedError as e:
        print(f"rep {rep}: FAILED {e.__cause__}", flush=True)
        bad += 1
        break
    dt = time.time() - t0
    res = verify.cholesky_residual(A, M.tiles, n, b)
    st = [eng.stats(d) for d in range(len(ords))]
    print(f"rep {rep}: {dt:.3f} s residual {res:.3e} p2p {sum(s['bytes_p2p_in'] for s in st) / 2**30:.2f} GiB "
          f"viol {eng.violations()}", flush=True)
    bad += res > verify.CHOL_RESIDUAL_TOL
eng.stop()
print("BAD" if bad else "OK", bad)
