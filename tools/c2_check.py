"""Debug: C2 full size, check every C tile against cuBLAS (torch fp64 on GPU)."""
import os, sys, time, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import torch
import paper_2308_15964_b200 as sf
from paper_2308_15964_b200 import algorithms as alg

n = int(os.environ.get("N", 16384)); b = int(os.environ.get("B", 512))
streams = int(os.environ.get("STREAMS", 32)); group = int(os.environ.get("GROUP", 32))
steps = int(os.environ.get("STEPS", 1))
gated = os.environ.get("GATED", "0") == "1"
nt = n // b
eng = sf.create_engine(sf.WorkerTeam.of_devices(1, streams), scheduler="prio", trace=False, group_max=group,
                       device_memory=24 << 30)
A, B, C = (alg.TiledMatrix(n, b) for _ in range(3))
g = sf.TaskGraph().compute_on(eng)
alg.insert_fill_uniform(g, A, 1); alg.insert_fill_uniform(g, B, 2); alg.insert_zero(g, C)
g.wait_all()
p0 = sf.gemm_paths()
t0 = time.time()
for _ in range(steps):
    if gated:
        with g.gated():
            alg.insert_gemm(g, A, B, C)
    else:
        alg.insert_gemm(g, A, B, C)
g.flush_all(keep_device=True)
g.wait_all()
p1 = sf.gemm_paths()
print("paths", {k: p1[k] - p0[k] for k in p1}, "t", time.time() - t0, flush=True)
eng.stop()
dev = torch.device("cuda")
def dense(M):
    return torch.from_numpy(M.to_dense()).to(dev)
Ad, Bd, Cd = dense(A), dense(B), dense(C)
want = (Ad @ Bd) * steps
err = (Cd - want).abs() / want.abs()
bad = err > 1e-10
print("max rel", err.max().item(), "bad elems", int(bad.sum().item()), flush=True)
if bad.any():
    tb = bad.reshape(nt, b, nt, b).any(dim=3).any(dim=1)
    idx = tb.nonzero().tolist()
    print("bad tiles", len(idx), idx[:40])
    for (i, j) in idx[:6]:
        tile_bad = bad[i*b:(i+1)*b, j*b:(j+1)*b]
        rows = tile_bad.any(dim=1).nonzero().flatten().tolist()
        cols = tile_bad.any(dim=0).nonzero().flatten().tolist()
        d = (Cd - want)[i*b:(i+1)*b, j*b:(j+1)*b]
        print(f"tile {i},{j}: nbad {int(tile_bad.sum())} rows {rows[:5]}..{rows[-3:]} ({len(rows)}) cols {cols[:5]}..{cols[-3:]} ({len(cols)}) maxabs {d.abs().max().item():.3g}")
        # express the error in units of one k-tile product
        for k in range(nt):
            pk = Ad[i*b:(i+1)*b, k*b:(k+1)*b] @ Bd[k*b:(k+1)*b, j*b:(j+1)*b]
            r = (d + pk).abs().max().item()
            if r < 1e-6 * pk.abs().max().item():
                print(f"   = minus exactly k-product {k}")
            r2 = (d - pk).abs().max().item()
            if r2 < 1e-6 * pk.abs().max().item():
                print(f"   = plus exactly k-product {k}")
