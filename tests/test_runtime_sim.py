"""The native runtime's bookkeeping on the simulated backend (no GPU).

The same libsfx.so that drives the B200s runs here against host-memory
devices (the reference's own simulated-device design), so its
dependency core, scheduler order, LRU arena and coherency are checked against
the golden fixtures produced by the real reference.  Only runtime test ops
execute in sim mode; tile ops are refused (test_native_abi.py).
"""

import json
import os
import random

import numpy as np
import pytest

import paper_2308_15964_b200 as sf
from oracle import programs

GOLD = os.path.join(os.path.dirname(__file__), "golden")
MODE = {"read": sf.read, "write": sf.write, "atomic": sf.atomic_write, "commute": sf.commutative_write,
        "maybe": sf.maybe_write}


def sim_engine(devices=1, streams=1, sched=None, **kw):
    return sf.create_engine(sf.WorkerTeam.of_devices(devices, streams), scheduler=sched, backend="sim", **kw)


def insert_program(g, prog):
    cells = [sf.Cell(i + 1) for i in range(prog["n_cells"])]
    tids = []
    for mode, target, reads, a, b in prog["tasks"]:
        acc = [MODE[mode](cells[target])] + [sf.read(cells[r]) for r in reads]
        tids.append(g.task(*acc, device=sf.ops.cell(mode, a, b)).task_id)
    return cells, tids


def pop_indices(g, tids):
    index = {t: i for i, t in enumerate(tids)}
    return [index[e[3]] for e in g.trace.export_events() if e[0] == "Pop" and e[3] in index]


def edge_indices(g, tids):
    index = {t: i for i, t in enumerate(tids)}
    return sorted({(index[s], index[d]) for s, d, _ in g.edges() if s in index and d in index})


@pytest.fixture(scope="module")
def random_programs():
    with open(os.path.join(GOLD, "random_programs.json")) as fh:
        return json.load(fh)


def test_random_programs_gated_match_reference(random_programs):
    eng = sim_engine()
    try:
        for p in random_programs:
            g = sf.TaskGraph().compute_on(eng)
            with g.gated():
                cells, tids = insert_program(g, p)
            for c in cells:
                g.flush_to_host(c)
            assert g.wait_all(timeout=30)
            assert [c.value for c in cells] == p["sequential"]
            assert edge_indices(g, tids) == sorted(tuple(e) for e in p["edges"])
            assert pop_indices(g, tids) == p["pop_order"]
    finally:
        eng.stop()


@pytest.mark.parametrize("devices,streams", [(1, 2), (1, 8), (2, 1), (4, 2)])
def test_random_programs_serial_equivalence(random_programs, devices, streams):
    eng = sim_engine(devices, streams)
    try:
        for p in random_programs:
            g = sf.TaskGraph().compute_on(eng)
            cells, _ = insert_program(g, p)
            for c in cells:
                g.flush_to_host(c)
            assert g.wait_all(timeout=30)
            assert [c.value for c in cells] == p["sequential"]
    finally:
        eng.stop()


@pytest.mark.parametrize("name,prog", [
    ("gemm_nt8", programs.gemm_program(8)),
    ("cholesky_nt8", programs.cholesky_program(8)),
    ("cholesky_nt32", programs.cholesky_program(32)),
    ("particles_g16", programs.particles_program(16)),
])
def test_tile_graphs_gated_match_reference(name, prog):
    gold = np.load(os.path.join(GOLD, "tile_graphs.npz"))
    eng = sim_engine()
    try:
        g = sf.TaskGraph().compute_on(eng)
        objs = {}
        tids = []
        with g.gated():
            for kind, acc, _ in prog:
                specs = []
                for mode, key in acc:
                    if key not in objs:
                        objs[key] = np.zeros(1)
                    specs.append({"read": sf.read, "write": sf.write,
                                  "commutative_write": sf.commutative_write}[mode](objs[key]))
                tids.append(g.task(*specs, device=sf.ops.noop, name=kind).task_id)
        assert g.wait_all(timeout=60)
        assert edge_indices(g, tids) == sorted(map(tuple, gold[f"{name}_edges"].tolist()))
        assert pop_indices(g, tids) == gold[f"{name}_pop"].tolist()
    finally:
        eng.stop()


def test_lru_matches_reference_arena():
    with open(os.path.join(GOLD, "lru.json")) as fh:
        cases = json.load(fh)
    for c in cases[:120]:
        eng = sim_engine(device_memory=c["capacity"], arena_align=8)
        try:
            g = sf.TaskGraph().compute_on(eng)
            bufs = [bytearray([h % 256] * c["size"]) for h in range(12)]
            hid = {}
            for h, b in enumerate(bufs):
                hid[g.register(b)] = h
            for h, want in zip(c["seq"], c["resident"]):
                g.task(sf.read(bufs[h]), device=sf.ops.noop)
                assert g.wait_all(timeout=10)
                assert sorted(hid[x] for x in eng.resident(0)) == want
        finally:
            eng.stop()


def test_restaging_unmodified_data_moves_nothing():
    # reference tests/test_device.py:161-177 and criterion 5
    eng = sim_engine()
    try:
        g = sf.TaskGraph().compute_on(eng)
        buf = bytearray(range(64))
        g.task(sf.read(buf), device=sf.ops.noop)
        g.wait_all(timeout=10)
        assert eng.stats(0)["bytes_to_device"] == 64
        g.task(sf.read(buf), device=sf.ops.noop)
        g.wait_all(timeout=10)
        assert eng.stats(0)["bytes_to_device"] == 64
        assert eng.stats(0)["hits"] == 1
    finally:
        eng.stop()


def test_host_coherency_round_trip():
    # reference tests/test_device.py:180-207 (host reads go through an explicit flush)
    eng = sim_engine()
    try:
        g = sf.TaskGraph().compute_on(eng)
        buf = bytearray(16)
        g.task(sf.write(buf), device=sf.ops.bytes_add(0, 16, 7))
        g.wait_all(timeout=10)
        hid = g.hid_of(buf)
        st = eng.block_state(hid, 0)
        assert st["dirty"] and not st["host_valid"]
        assert buf == bytearray(16)  # host copy is stale until flushed
        g.flush_to_host(buf)
        g.wait_all(timeout=10)
        assert buf == bytearray([7] * 16)
        assert not eng.block_state(hid, 0)["present"]  # host write drops device copies
        before = eng.stats(0)["bytes_to_device"]
        g.task(sf.write(buf), device=sf.ops.bytes_add(0, 1, 1))
        g.flush_to_host(buf, keep_device=True)
        g.wait_all(timeout=10)
        assert buf[0] == 8
        assert eng.stats(0)["bytes_to_device"] == before + 16
        st = eng.block_state(hid, 0)
        assert st["valid"] and not st["dirty"] and st["host_valid"]
    finally:
        eng.stop()


def _random_byte_program(rng):
    # reference tests/test_acceptance.py:225-236
    bufs = [bytearray(rng.randrange(256) for _ in range(rng.choice((16, 24, 32)))) for _ in range(rng.randint(2, 4))]
    ops = []
    for _ in range(rng.randint(4, 12)):
        b = rng.randrange(len(bufs))
        size = len(bufs[b])
        off = rng.randrange(size)
        length = rng.randint(1, size - off)
        ops.append((b, off, length, rng.randint(1, 255)))
    return bufs, ops


def test_tiny_arena_round_trips_match_host_execution():
    # criterion 5: 100 random byte programs through a 64-byte arena (forced eviction)
    rng = random.Random(5)
    eng = sim_engine(device_memory=64, arena_align=8)
    try:
        for _ in range(100):
            bufs, ops = _random_byte_program(rng)
            expected = [bytearray(b) for b in bufs]
            for b, off, length, delta in ops:
                for i in range(off, off + length):
                    expected[b][i] = (expected[b][i] + delta) % 256
            g = sf.TaskGraph().compute_on(eng)
            for b, off, length, delta in ops:
                g.task(sf.write(bufs[b]), device=sf.ops.bytes_add(off, length, delta))
            for b in bufs:
                g.flush_to_host(b)
            assert g.wait_all(timeout=30)
            assert bufs == expected
        assert eng.stats(0)["evictions"] > 0
    finally:
        eng.stop()


def test_pinned_exhaustion_poisons_cleanly():
    # reference tests/test_device.py:255-263
    eng = sim_engine(device_memory=64, arena_align=8)
    try:
        g = sf.TaskGraph().compute_on(eng)
        a, b = bytearray(48), bytearray(48)
        g.task(sf.read(a), sf.read(b), device=sf.ops.noop)
        with pytest.raises(sf.EngineFailedError) as info:
            g.wait_all(timeout=10)
        assert isinstance(info.value.__cause__, sf.StagingError)
        assert "pinned" in str(info.value.__cause__)
    finally:
        eng.stop()


def test_oversized_object_rejected():
    eng = sim_engine(device_memory=16, arena_align=8)
    try:
        g = sf.TaskGraph().compute_on(eng)
        g.task(sf.read(bytearray(32)), device=sf.ops.noop)
        with pytest.raises(sf.EngineFailedError) as info:
            g.wait_all(timeout=10)
        assert isinstance(info.value.__cause__, sf.StagingError)
        assert "exceeds" in str(info.value.__cause__)
    finally:
        eng.stop()


def test_cross_device_reads_pull_peer_to_peer():
    """Deliberate divergence from reference tests/test_device.py:210-236: the
    freshest copy moves device -> device (NVLink) and the host stays stale."""
    eng = sim_engine(devices=2)
    try:
        g = sf.TaskGraph().compute_on(eng)
        buf = bytearray(32)
        g.task(sf.write(buf), device=sf.ops.bytes_add(0, 4, 9), priority=0)
        g.wait_all(timeout=10)
        hid = g.hid_of(buf)
        owner = 0 if eng.block_state(hid, 0)["dirty"] else 1
        other = 1 - owner
        # force the reader onto the other device
        g._submit_one(9_000_000_001, sf.ops.noop, 0, [hid], [0], dev_hint=other)
        g.wait_all(timeout=10)
        assert eng.stats(other)["bytes_p2p_in"] == 32
        assert eng.stats(other)["bytes_to_device"] == 0
        assert eng.block_state(hid, owner)["dirty"]          # owner keeps the single dirty copy
        assert eng.block_state(hid, other)["valid"]
        assert not eng.block_state(hid, owner)["host_valid"]  # host not touched
        # a writer on `other` invalidates the owner's copy
        g._submit_one(9_000_000_002, sf.ops.bytes_add(0, 1, 1), 0, [hid], [1], dev_hint=other)
        g.wait_all(timeout=10)
        assert not eng.block_state(hid, owner)["present"]
        assert eng.block_state(hid, other)["dirty"]
        g.flush_to_host(buf)
        g.wait_all(timeout=10)
        assert buf[:4] == bytearray([10, 9, 9, 9])
    finally:
        eng.stop()


def test_priority_scheduler_pops_in_priority_order():
    rng = random.Random(99)
    eng = sim_engine(sched="prio")
    try:
        for _ in range(30):
            g = sf.TaskGraph().compute_on(eng)
            prios = [rng.randint(-50, 50) for _ in range(rng.randint(2, 30))]
            tids = []
            with g.gated():
                for p in prios:
                    tids.append(g.task(sf.write(sf.Cell(0)), device=sf.ops.noop, priority=p).task_id)
            assert g.wait_all(timeout=10)
            order = pop_indices(g, tids)
            popped = [prios[i] for i in order]
            assert all(a >= b for a, b in zip(popped, popped[1:]))
            # FIFO among equal priorities (scheduler.py:111)
            for a, b in zip(order, order[1:]):
                if prios[a] == prios[b]:
                    assert a < b
    finally:
        eng.stop()


def test_wait_all_timeout_and_resume():
    eng = sim_engine()
    try:
        g = sf.TaskGraph().compute_on(eng)
        eng.pause()
        c = sf.Cell(1)
        g.task(sf.write(c), device=sf.ops.cell("write", 2, 0))
        assert g.wait_all(timeout=0.2) is False
        eng.resume()
        assert g.wait_all(timeout=10) is True
    finally:
        eng.stop()


def test_runtime_options_and_kernel_timing_toggle():
    eng = sim_engine(kernel_timing=True)
    try:
        for key, val in (("group_max", 8), ("groups_per_stream", 4), ("prefetch", 0), ("prefetch_depth", 16),
                         ("window", 256), ("urgent_priority", 10), ("kernel_timing", 0), ("kernel_timing", 1)):
            eng.set_option(key, val)
        with pytest.raises(sf.ConfigurationError):
            eng.set_option("no_such_knob", 1)
        g = sf.TaskGraph().compute_on(eng)
        c = sf.Cell(1)
        for _ in range(4):
            g.task(sf.commutative_write(c), device=sf.ops.cell("commute", 1, 1))
        eng.set_option("kernel_timing", 0)
        for _ in range(4):
            g.task(sf.commutative_write(c), device=sf.ops.cell("commute", 1, 1))
        g.flush_all()  # flush tasks are asynchronous like every task
        g.wait_all()
        assert c.value == 9
    finally:
        eng.stop()


def test_insertion_errors_match_reference():
    eng = sim_engine()
    try:
        g = sf.TaskGraph()
        with pytest.raises(sf.ConfigurationError):
            g.task(sf.write(sf.Cell(0)), device=sf.ops.noop)  # not attached
        g.compute_on(eng)
        with pytest.raises(sf.ConfigurationError):
            g.compute_on(eng)
        c = sf.Cell(0)
        with pytest.raises(sf.DuplicateAccessError):
            g.task(sf.read(c), sf.write(c), device=sf.ops.noop)
        with pytest.raises(sf.ConfigurationError, match="oracle"):
            g.task(sf.write(c), host=lambda x: None)
        with pytest.raises(sf.ConfigurationError):
            g.task(sf.write(c), device=42)  # neither an op nor a callable (callables are user ops)
        with pytest.raises(sf.ConfigurationError):
            g.task(sf.write(c))
        with pytest.raises(sf.ConfigurationError):
            g.task("not an access", device=sf.ops.noop)
        with pytest.raises(sf.SpeculationError):
            sf.TaskGraph(speculation=True)
        assert g.wait_all(timeout=5)
    finally:
        eng.stop()


def test_dot_dialect_matches_reference_parser():
    # reference tests/conftest.py:206-226
    import re

    node = re.compile(r"^  t(\d+) \[(.*)\];$")
    edge = re.compile(r"^  t(\d+) -> t(\d+)(?: \[label=(.*)\])?;$")
    eng = sim_engine()
    try:
        g = sf.TaskGraph().compute_on(eng)
        a, b = sf.Cell(1), sf.Cell(2)
        t1 = g.task(sf.write(a), device=sf.ops.noop, name='first "q"')
        t2 = g.task(sf.read(a), sf.write(b), device=sf.ops.noop)
        g.wait_all(timeout=5)
        for show in (False, True):
            lines = g.generate_dot(show_deps=show).strip().splitlines()
            assert lines[0] == "digraph taskgraph {" and lines[-1] == "}"
            edges = []
            for line in lines[1:-1]:
                if node.match(line):
                    continue
                m = edge.match(line)
                assert m, line
                edges.append((int(m.group(1)), int(m.group(2))))
            assert edges == [(t1.task_id, t2.task_id)]
    finally:
        eng.stop()


def test_trace_has_four_events_per_task_and_push_precedes_pop():
    # reference tests/test_trace.py:116-139
    eng = sim_engine(streams=2)
    try:
        g = sf.TaskGraph().compute_on(eng)
        cells = [sf.Cell(i) for i in range(4)]
        for i in range(40):
            g.task(sf.write(cells[i % 4]), sf.read(cells[(i + 1) % 4]), device=sf.ops.noop)
        g.wait_all(timeout=10)
        ev = g.trace.export_events()
        per = {}
        for kind, t, wid, tid, _ in ev:
            per.setdefault(tid, {})[kind] = t
        assert len(per) == 40
        for tid, kinds in per.items():
            assert set(kinds) == {"Push", "Pop", "TaskStart", "TaskEnd"}
            assert kinds["Push"] <= kinds["Pop"] <= kinds["TaskStart"] <= kinds["TaskEnd"]
        svg = g.generate_trace_svg()
        assert svg.startswith("<svg")
        assert eng.violations() == 0
    finally:
        eng.stop()


def test_cell_semantics():
    c = sf.Cell(3)
    assert c.value == 3 and c == sf.Cell(3) and c != sf.Cell(3.0)
    f = sf.Cell(1.5)
    f.value = 2.5
    assert f.value == 2.5
    with pytest.raises(TypeError):
        f.value = 1
    b = sf.Cell(True)
    assert b.value is True


def test_cholesky_priorities_match_oracle_program():
    from paper_2308_15964_b200.algorithms import cholesky_priorities as P

    for nt in (2, 5, 8):
        prog = programs.cholesky_program(nt)
        mine = []
        for k in range(nt):
            mine.append(P(nt, "potrf", k))
            for i in range(k + 1, nt):
                mine.append(P(nt, "trsm", k, i))
            for i in range(k + 1, nt):
                mine.append(P(nt, "syrk", k, i))
                for j in range(k + 1, i):
                    mine.append(P(nt, "gemm", k, i, j))
        assert mine == [p for _, _, p in prog]


def test_block_cyclic_owner_computes_on_simulated_devices():
    """Every task runs on the device that owns (home) the tile it writes; reads
    of remote tiles arrive peer-to-peer; the dependency edges are the oracle's."""
    from paper_2308_15964_b200 import algorithms as alg

    nt, ndev = 6, 4
    eng = sim_engine(devices=ndev, streams=2)
    try:
        g = sf.TaskGraph().compute_on(eng)
        tiles = {(i, j): np.zeros(4) for i in range(nt) for j in range(i + 1)}
        P, Q = alg.grid_shape(ndev)
        owner = {ij: (ij[0] % P) * Q + (ij[1] % Q) for ij in tiles}
        for ij, t in tiles.items():
            g.place(t, owner[ij])
        prog = programs.cholesky_program(nt)
        tids, out_tile = [], {}
        with g.gated():  # static slot layout, comparable with the oracle's edges
            for kind, acc, prio in prog:
                specs = [{"read": sf.read, "write": sf.write}[m](tiles[key[1:]]) for m, key in acc]
                t = g.task(*specs, device=sf.ops.noop, priority=prio, name=kind)
                tids.append(t.task_id)
                out_tile[t.task_id] = [key[1:] for m, key in acc if m == "write"][0]
        assert g.wait_all(timeout=60)
        k = eng.streams_per_device
        streams = k + (max(2, k // 4) if k >= 2 else 0)  # normal + urgent streams per device (sim: no coop)
        pops = {tid: wid for kind, _, wid, tid, _ in g.trace.export_events() if kind == "Pop"}
        for tid in tids:
            dev = pops[tid] // streams
            assert dev == owner[out_tile[tid]], (tid, dev, owner[out_tile[tid]])
        assert sum(eng.stats(d)["copies_p2p_in"] for d in range(ndev)) > 0
        want = stf_edges(prog)
        assert edge_indices(g, tids) == sorted(want)
    finally:
        eng.stop()


def stf_edges(prog):
    from oracle import stf

    return stf.static_successor_edges(programs.program_accesses(prog))


@pytest.mark.parametrize("devices,streams", [(1, 4), (2, 3)])
def test_shared_commutative_guard_mixed_with_exclusive_members(devices, streams):
    """Ops that accumulate with device atomics (add_i64, the P2P ops) take the
    commutative guard in shared mode; exclusive members of the same group (cell
    'commute') still exclude them.  Values equal a serial execution, and the
    commutative groups still produce no edges among their members."""
    rng = random.Random(7)
    n = 6
    eng = sim_engine(devices, streams)
    try:
        g = sf.TaskGraph().compute_on(eng)
        cells = [sf.Cell(0) for _ in range(n)]
        want = [0] * n
        for step in range(300):
            i, j = rng.sample(range(n), 2)
            if step % 50 == 49:  # a plain write closes the groups of cell i
                g.task(sf.write(cells[i]), sf.read(cells[j]), device=sf.ops.cell("write", 2, 1))
                want[i] = (2 * want[i] + 1 + want[j]) % 10000019  # reference tests/conftest.py:22
            elif rng.random() < 0.2:
                g.task(sf.commutative_write(cells[i]), device=sf.ops.cell("commute", 1, 3))
                want[i] = (want[i] + 3) % 10000019
            else:
                d = rng.randrange(1, 100)
                g.task(sf.commutative_write(cells[i]), sf.commutative_write(cells[j]), device=sf.ops.add_i64(d))
                want[i] += d
                want[j] += d
        assert g.wait_all(timeout=60)
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=60)
    finally:
        eng.stop()
    assert [c.value for c in cells] == want


def _submit_with_hints(g, op, cells_per_task, hints, mode=sf.AccessMode.ATOMIC_WRITE):
    import numpy as np

    n = len(cells_per_task)
    k = len(cells_per_task[0])
    hids = np.array([[g.hid_of(c) for c in row] for row in cells_per_task], np.uint64).reshape(-1)
    return g.submit_arrays(np.full(n, op.code, np.uint32), np.tile(np.array(op.fparam), (n, 1)),
                           np.tile(np.array(op.iparam, np.int64), (n, 1)), np.zeros(n, np.int32),
                           np.full(n, k, np.uint32), hids, np.full(n * k, mode.code, np.uint32),
                           devices=np.asarray(hints, np.int32))


def test_atomic_group_members_share_one_device_despite_hints():
    """members of one atomic slot run concurrently, so they must share
    one device copy.  The group's device (set by its first member) overrides
    later members' hints and the tiles' homes."""
    eng = sim_engine(2, 2)
    try:
        g = sf.TaskGraph().compute_on(eng)
        c = sf.Cell(0)
        g.place(c, 1)
        _submit_with_hints(g, sf.ops.add_i64(1), [[c]] * 40, [0, 1] * 20)
        g.flush_to_host(c)
        assert g.wait_all(timeout=30)
        assert c.value == 40
        assert eng.stats(0)["tasks_executed"] >= 40 and eng.stats(1)["tasks_executed"] == 0
    finally:
        eng.stop()


def test_atomic_members_joining_two_device_groups_serialise():
    """A member whose atomic handles belong to groups on different devices runs
    under the shared guards (never concurrently with the other device's members);
    the result equals the serial sum."""
    rng = random.Random(3)
    eng = sim_engine(2, 3)
    try:
        g = sf.TaskGraph().compute_on(eng)
        cells = [sf.Cell(0) for _ in range(4)]
        want = [0] * 4
        rows, hints = [], []
        for _ in range(400):
            i, j = rng.sample(range(4), 2)
            rows.append([cells[i], cells[j]])
            hints.append(rng.randrange(2))
            want[i] += 2
            want[j] += 2
        _submit_with_hints(g, sf.ops.add_i64(2), rows, hints)
        for c in cells:
            g.flush_to_host(c)
        assert g.wait_all(timeout=30)
        assert [c.value for c in cells] == want
    finally:
        eng.stop()


def test_random_programs_on_array_elements_match_reference(random_programs):
    """Array views (reference access.py:103-129): the reference's random programs
    with every cell an ELEMENT of one int64 array, accessed through
    write_array / read_array / commutative_write_array / ...  Each element is its
    own handle, so the dependency edges and the values equal the reference's for
    the same programs on separate cells (tests/golden/random_programs.json)."""
    amode = {"read": sf.read_array, "write": sf.write_array, "atomic": sf.atomic_write_array,
             "commute": sf.commutative_write_array, "maybe": sf.maybe_write_array}
    eng = sim_engine(1, 1)
    try:
        for p in random_programs[:60]:
            X = np.arange(1, p["n_cells"] + 1, dtype=np.int64)
            g = sf.TaskGraph().compute_on(eng)
            tids = []
            with g.gated():
                for m, target, reads, a, b in p["tasks"]:
                    acc = [amode[m](X, [target])]
                    if reads:
                        acc.append(sf.read_array(X, reads))
                    tids.append(g.task(*acc, device=sf.ops.cell(m, a, b)).task_id)
            assert g.wait_all(timeout=30)
            assert edge_indices(g, tids) == sorted(map(tuple, p["edges"]))
            for i in range(p["n_cells"]):
                g.flush_to_host(X, element=i)
            assert g.wait_all(timeout=30)
            assert X.tolist() == p["sequential"]
    finally:
        eng.stop()


def test_array_view_errors_and_whole_object_independence():
    eng = sim_engine(1, 1)
    try:
        g = sf.TaskGraph().compute_on(eng)
        X = np.zeros(4, np.int64)
        with pytest.raises(sf.DuplicateAccessError):
            sf.read_array(X, [1, 1])
        with pytest.raises(sf.DuplicateAccessError):
            g.task(sf.write_array(X, [2]), sf.read_array(X, [2]), device=sf.ops.noop)
        with pytest.raises(IndexError):
            g.task(sf.write_array(X, [7]), device=sf.ops.noop)
        # element handles are distinct from the whole-object handle (reference
        # registry keys (id(obj)) vs (id(obj), element)): no edge between them
        t1 = g.task(sf.write_array(X, [0]), device=sf.ops.cell("write", 2, 1)).task_id
        t2 = g.task(sf.write(X), device=sf.ops.noop).task_id
        assert g.wait_all(timeout=10)
        assert (t1, t2) not in {(s, d) for s, d, _ in g.edges()}
    finally:
        eng.stop()


def test_object_in_two_graphs_hands_over_through_the_host():
    """One live handle per host buffer across graphs: registering an object in a
    second graph retires the first graph's handle (its dirty device copy is
    written home first), so the second graph sees the first one's result; the
    first graph can no longer use the object; a busy object cannot move."""
    eng = sim_engine(2, 2)
    try:
        c = sf.Cell(5)
        g1 = sf.TaskGraph().compute_on(eng)
        g1.task(sf.write(c), device=sf.ops.cell("write", 3, 1))  # 16, dirty on a device
        assert g1.wait_all(timeout=10)
        g2 = sf.TaskGraph().compute_on(eng)
        g2.task(sf.write(c), device=sf.ops.cell("write", 2, 0))  # 2 * 16
        g2.flush_to_host(c)
        assert g2.wait_all(timeout=10)
        assert c.value == 32
        with pytest.raises(sf.RegistrationError):
            g1.task(sf.read(c), device=sf.ops.noop)
        # a busy object: g3 holds pending work on d (paused engine), g4 may not take it
        d = sf.Cell(1)
        g3 = sf.TaskGraph().compute_on(eng)
        eng.pause()
        try:
            g3.task(sf.write(d), device=sf.ops.cell("write", 1, 1))
            g4 = sf.TaskGraph().compute_on(eng)
            with pytest.raises(sf.RegistrationError):
                g4.task(sf.read(d), device=sf.ops.noop)
        finally:
            eng.resume()
        assert g3.wait_all(timeout=10)
    finally:
        eng.stop()


@pytest.mark.parametrize("devices,streams", [(1, 1), (2, 3)])
def test_history_free_graphs_retire_tasks_and_keep_semantics(random_programs, devices, streams):
    """TaskGraph(history=False): finished tasks and passed slots are retired
    (reference handles.py:114-189 retires handles; here the runtime's task/slot
    records go back to a pool) -- values still equal the sequential execution,
    and only the tasks of each handle's last slot stay live."""
    eng = sim_engine(devices, streams)
    try:
        for p in random_programs:
            g = sf.TaskGraph(history=False).compute_on(eng)
            cells, tids = insert_program(g, p)
            for c in cells:
                g.flush_to_host(c)
            assert g.wait_all(timeout=30)
            assert [c.value for c in cells] == p["sequential"]
            sf.TaskViewer(g, tids[0]).wait()  # a retired task reads as finished
        live = eng.live()
        assert live["retired"] > 0
    finally:
        eng.stop()


def test_million_task_soak_has_flat_runtime_memory():
    """10^6 tasks through one history-free graph: the live task and slot counts
    and the process RSS stay flat (round-1 review: task_store_/slots only grew)."""
    import psutil

    eng = sim_engine(1, 4)
    proc = psutil.Process()
    try:
        g = sf.TaskGraph(history=False, trace=False).compute_on(eng)
        T = 8
        cells = [sf.Cell(0) for _ in range(T)]
        H = np.array([g.hid_of(c) for c in cells], np.uint64)
        op = sf.ops.cell("write", 1, 1)
        chunk = 20000
        rss = []
        for rep in range(50):  # 50 x 20,000 = 10^6 tasks
            hids = np.tile(H, chunk // T)
            g.submit_arrays(np.full(chunk, op.code, np.uint32), np.zeros((chunk, 4)),
                            np.tile(np.array(op.iparam, np.int64), (chunk, 1)), np.zeros(chunk, np.int32),
                            np.ones(chunk, np.uint32), hids, np.full(chunk, sf.AccessMode.WRITE.code, np.uint32))
            assert g.wait_all(timeout=60)
            live = eng.live()
            assert live["tasks"] <= 2 * T and live["slots"] <= 2 * T, live
            rss.append(proc.memory_info().rss)
        g.flush_all(keep_device=False)
        assert g.wait_all(timeout=60)
        assert eng.live()["retired"] >= 10 ** 6 - 2 * T
        assert [c.value for c in cells] == [(10 ** 6 // T)] * T  # x <- x + 1 per task
        assert rss[-1] - rss[5] < 32 << 20, (rss[5], rss[-1])
    finally:
        eng.stop()
