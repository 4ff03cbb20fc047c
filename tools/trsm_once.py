"""One POTRF(full inverse) + TRSM(full inverse) pair at b (default 1024), run twice:
the target for ncu captures of potrf_flow_kernel and of the TRI-masked DGEMM."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_15964_b200 as sf  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 4), trace=False)
g = sf.TaskGraph().compute_on(eng)
L = sf.pinned_empty((b, b))
B = sf.pinned_empty((b, b))
for _ in range(2):
    g.task(sf.write(L), device=sf.ops.fill_spd(51, 0, 0, b))
    g.task(sf.write(B), device=sf.ops.fill_uniform(52, 0, 0, b))
    g.task(sf.write(L), device=sf.ops.potrf_fullinv)
    g.task(sf.read(L), sf.write(B), device=sf.ops.trsm_fullinv)
    g.wait_all()
eng.stop()
print("ok")
