"""The reference overhead protocol (bench.overhead_gpu) on the GPU engine for a
few configurations; prints one line per configuration.

    python tools/overhead_probe.py [T] [N]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2308_15964_b200 as sf  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else (os.cpu_count() or 4)
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
for D, mode, deps in ((0.0, "write", 1), (1e-4, "write", 1), (1e-3, "write", 1), (1e-3, "commute", 1),
                      (1e-4, "write", 20)):
    r = bench.overhead_gpu(sf, 0, T, N, D, mode, deps, reps=2)
    print(f"D={D:g} {mode} deps={deps}: " + " ".join(f"{k}={v:.2f}" for k, v in r.items()), flush=True)
