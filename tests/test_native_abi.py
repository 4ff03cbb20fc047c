"""The C-ABI library loads, exports every symbol include/sfx.h declares, and its
structs match the Python binding.  No compute calls (runs without a GPU)."""

import ctypes
import os
import re
import subprocess

import pytest

import paper_2308_15964_b200 as sf
from paper_2308_15964_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sfx.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sfx_\w+)\s*\(", text, re.M)))


def test_header_declares_the_abi():
    names = declared_functions()
    assert "sfx_create" in names and "sfx_submit" in names and "sfx_wait_all" in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(N.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared_functions()) == set(N.EXPORTED)


def test_exported_symbols_are_c_linkage():
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True).stdout
    syms = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for name in declared_functions():
        assert name in syms, f"{name} not exported with C linkage"


def test_struct_layouts():
    assert ctypes.sizeof(N.TaskDesc) == 96
    assert ctypes.sizeof(N.AccessDesc) == 16
    assert ctypes.sizeof(N.Event) == 32
    text = open(HEADER).read()
    body = text[text.index("typedef struct sfx_dev_stats"):text.index("} sfx_dev_stats;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"(\w+)\s*[,;]", body.split("{", 1)[1])
    assert len(fields) == len(N.DevStats._fields_)


def test_abi_version_and_device_count():
    assert N.lib.sfx_abi_version() == 1
    assert sf.device_count() >= 0


def test_cuda_engine_fails_loudly_without_gpu():
    if sf.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(sf.ConfigurationError):
        sf.create_engine(sf.WorkerTeam.of_devices(1, 1))


def test_sim_refuses_tile_ops():
    eng = sf.create_engine(sf.WorkerTeam.of_devices(1, 1), backend="sim")
    try:
        g = sf.TaskGraph().compute_on(eng)
        import numpy as np

        a, b, c = (np.zeros((64, 64)) for _ in range(3))
        with pytest.raises(sf.ConfigurationError, match="CUDA device"):
            g.task(sf.read(a), sf.read(b), sf.write(c), device=sf.ops.gemm_nn)
    finally:
        eng.stop()


def test_kernels_compiled_for_sm100a():
    out = subprocess.run(["cuobjdump", "-lelf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_dgemm_uses_dmma_and_tma():
    out = subprocess.run(["cuobjdump", "-sass", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "DMMA.8x8x4" in out.stdout
    assert "UTMALDG" in out.stdout
