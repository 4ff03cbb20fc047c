"""The N>1 launch path on CPU: torchrun with world_size 2 over gloo (127.0.0.1).

bench.py's per-rank plumbing (Dist: barrier, max over ranks) and the reference
arm's rank discipline (rank 0 alone runs and prints ONE JSON line; the other
ranks exit 0 without work) are what the driver relies on at N > 1.
"""

import json
import os
import re
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _json_lines(text):
    """Flat JSON objects printed by the ranks (two ranks' lines may interleave in
    the captured stream, so objects are matched rather than lines)."""
    return [json.loads(m) for m in re.findall(r"\{[^{}]*\}", text)]


def _torchrun(args, timeout=240):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port())] + args
    env = dict(os.environ, OMP_NUM_THREADS="1")
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def test_dist_max_over_ranks_gloo(tmp_path):
    script = tmp_path / "ranks.py"
    script.write_text(
        "import json, os, sys\n"
        f"sys.path.insert(0, {ROOT!r})\n"
        "import bench\n"
        "d = bench.Dist()\n"
        "d.init('gloo')\n"
        "d.barrier()\n"
        "m = d.max(float(d.rank + 1) * 1.5)\n"
        "print(json.dumps({'rank': d.rank, 'world': d.world, 'max': m}), flush=True)\n"
        "d.done()\n")
    r = _torchrun([str(script)])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert sorted(x["rank"] for x in lines) == [0, 1]
    assert all(x["world"] == 2 and x["max"] == 3.0 for x in lines)


def test_reference_arm_prints_once_under_torchrun():
    r = _torchrun(["bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
                   "--matrix-n", "1024", "--tile-b", "256", "--cpu-seconds", "0.5"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]  # rank 0 alone prints
    assert len(lines) == 1, r.stdout
    line = lines[0]
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "GFLOP/s"
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0


def test_comm_tasks_between_two_processes():
    """send / recv / broadcast tasks (reference comms.py, tests/test_comms.py) between
    two processes, each with its own native runtime: every tier, dependency
    ordering through a device task, FIFO matching on one tag, broadcast, a size
    mismatch poisoning with CommProtocolError, insertion validation."""
    r = _torchrun([os.path.join("tests", "dist", "comm_ranks.py")])
    assert r.returncode == 0, r.stderr[-3000:]
    out = {x["rank"]: x for x in _json_lines(r.stdout)}
    assert set(out) == {0, 1}
    for rank in (0, 1):
        assert out[rank]["tiers"] == [41, "ping", 66.0]
        assert out[rank]["dep"] == 16
        assert out[rank]["bcast"] == 777
        assert out[rank]["validation"] == ["config", "config", "config", "serialization"]
    assert out[1]["fifo"] == [1, 2, 3]
    assert out[0]["swap"] == 11.0 and out[1]["swap"] == 10.0
    assert out[1]["mismatch"] == "CommProtocolError"


@pytest.mark.gpu
def test_comm_tasks_with_gpu_engines():
    r = _torchrun([os.path.join("tests", "dist", "comm_gpu_ranks.py")])
    assert r.returncode == 0, r.stderr[-3000:]
    out = {x["rank"]: x for x in _json_lines(r.stdout)}
    assert out[0]["d2h"] >= 256 * 256 * 8  # the dirty GPU tile was fetched home before the send
    assert out[1]["recv_exact"] and out[1]["gemm_err"] <= 1e-15
