"""Run under torchrun (2 ranks, gloo): communication tasks between two graph
instances in two processes, each on its own native runtime (simulated
backend: no GPU needed).  Prints one JSON line per rank with what it saw."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2308_15964_b200 as sf  # noqa: E402

dist.init_process_group("gloo")
rank = dist.get_rank()
comm = sf.TorchComm()
out = {"rank": rank}
eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 2), backend="sim")
try:
    g = sf.TaskGraph().compute_on(eng).use_comm(comm)
    # 1. each tier: Cell, bytearray, numpy tile
    if rank == 0:
        c, b, t = sf.Cell(41), bytearray(b"ping"), np.arange(12, dtype=np.float64).reshape(3, 4)
        g.send(c, dest=1, tag=0)
        g.send(b, dest=1, tag=1)
        g.send(t, dest=1, tag=2)
    else:
        c, b, t = sf.Cell(0), bytearray(4), np.zeros((3, 4))
        g.recv(c, src=0, tag=0)
        g.recv(b, src=0, tag=1)
        g.recv(t, src=0, tag=2)
    assert g.wait_all(timeout=30)
    out["tiers"] = [c.value, bytes(b).decode(), float(t.sum())]
    # 2. a received value feeds a device task (ordering by dependency), and a
    #    device-written value is fetched home before it is sent
    if rank == 0:
        x = sf.Cell(5)
        g.task(sf.write(x), device=sf.ops.cell("write", 3, 1))  # x = 3*5 + 1 = 16 on the device
        g.send(x, dest=1, tag=3)
    else:
        x = sf.Cell(0)
        y = sf.Cell(0)
        g.recv(x, src=0, tag=3)
        g.task(sf.write(y), sf.read(x), device=sf.ops.cell("write", 1, 0))  # y = y + x
        g.flush_to_host(y)
    assert g.wait_all(timeout=30)
    out["dep"] = x.value if rank == 0 else y.value
    # 3. same tag: FIFO matching
    if rank == 0:
        for v in (1, 2, 3):
            g.send(sf.Cell(v), dest=1, tag=4)
        outs = []
    else:
        outs = [sf.Cell(0) for _ in range(3)]
        for o in outs:
            g.recv(o, src=0, tag=4)
    assert g.wait_all(timeout=30)
    out["fifo"] = [o.value for o in outs]
    # 4. broadcast from rank 1
    bc = sf.Cell(777 if rank == 1 else 0)
    g.broadcast(bc, root=1)
    assert g.wait_all(timeout=30)
    out["bcast"] = bc.value
    # 5. size mismatch poisons with CommProtocolError as the cause
    g2 = sf.TaskGraph().compute_on(sf.create_engine(sf.WorkerTeam.of_devices(1, 1), backend="sim")).use_comm(comm)
    if rank == 0:
        g2.send(bytearray(16), dest=1, tag=5)
        ok = g2.wait_all(timeout=30)
        out["mismatch"] = "sent" if ok else "timeout"
    else:
        g2.recv(bytearray(8), src=0, tag=5)
        try:
            g2.wait_all(timeout=30)
            out["mismatch"] = "no error"
        except sf.EngineFailedError as exc:
            out["mismatch"] = type(exc.__cause__).__name__
    g2.engine.stop()
    # 6. ADVICE r1: send(X) then recv(X) on the SAME buffer on both ranks (a swap):
    #    sends complete once posted (payload staged), so the recv behind each
    #    send can run and the exchange does not deadlock
    sw = np.full(6, float(10 + rank))
    g.send(sw, dest=1 - rank, tag=6)
    g.recv(sw, src=1 - rank, tag=6)
    g.task(sf.write(sw), device=sf.ops.noop)
    assert g.wait_all(timeout=30)
    out["swap"] = float(sw[0])
    # 7. insertion validation
    errs = []
    for kw in ({"dest": 5, "tag": 0}, {"dest": 1 - rank, "tag": -1}, {"dest": 1 - rank, "tag": 1 << 30}):
        try:
            g.send(sf.Cell(1), **kw)
        except sf.ConfigurationError:
            errs.append("config")
    try:
        g.send(object(), dest=1 - rank, tag=0)
    except sf.SerializationError:
        errs.append("serialization")
    out["validation"] = errs
finally:
    eng.stop()
print(json.dumps(out), flush=True)
dist.barrier()
dist.destroy_process_group()
