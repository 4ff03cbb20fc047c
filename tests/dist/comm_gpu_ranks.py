"""torchrun, 2 ranks (gloo), both on cuda:0: rank 0 generates a tile on the GPU
and sends it (the runtime fetches the dirty device copy home first); rank 1
receives it into a host tile and uses it in a GPU DGEMM (staged from the
received host buffer).  Prints one JSON line per rank."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2308_15964_b200 as sf  # noqa: E402
from oracle import inputs  # noqa: E402

dist.init_process_group("gloo")
rank = dist.get_rank()
comm = sf.TorchComm()
b = 256
eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 2), device_memory=1 << 30, ordinals=[0])
out = {"rank": rank}
try:
    g = sf.TaskGraph().compute_on(eng).use_comm(comm)
    A = sf.pinned_empty((b, b))
    if rank == 0:
        g.task(sf.write(A), device=sf.ops.fill_uniform(7, 0, 0, b))  # generated on the GPU
        g.send(A, dest=1, tag=0)
        assert g.wait_all(timeout=60)
    else:
        I = np.eye(b)
        C = sf.pinned_zeros((b, b))
        g.recv(A, src=0, tag=0)
        g.task(sf.read(A), sf.read(I), sf.write(C), device=sf.ops.gemm_nn)  # C += A I on the GPU
        g.flush_to_host(C)
        assert g.wait_all(timeout=60)
        want = inputs.uniform_tile(7, 0, 0, b, b, b)
        out["recv_exact"] = bool(np.array_equal(A, want))
        out["gemm_err"] = float(np.abs(C - want).max())
    out["d2h"] = eng.stats(0)["bytes_from_device"]
finally:
    eng.stop()
print(json.dumps(out), flush=True)
dist.barrier()
dist.destroy_process_group()
