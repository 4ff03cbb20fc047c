"""In-tree build of libsfx.so (the C-ABI runtime + sm_100a kernels).

``python -m paper_2308_15964_b200.build`` compiles every source under
``csrc/`` with nvcc for ``-gencode arch=compute_100a,code=sm_100a`` and links
``paper_2308_15964_b200/libsfx.so`` (static cudart, so the library loads on a
machine without a GPU; it only needs the driver when a CUDA runtime is
created).  Objects are cached in ``build/`` and rebuilt when a source or any
header is newer.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libsfx.so")
OBJDIR = os.path.join(ROOT, "build", "sfx")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libsfx.so")


def _sources():
    out = []
    for dirpath, _, files in os.walk(CSRC):
        for f in sorted(files):
            if f.endswith((".cu", ".cpp")):
                out.append(os.path.join(dirpath, f))
    return sorted(out)


def _headers():
    hs = [os.path.join(ROOT, "include", "sfx.h")]
    for dirpath, _, files in os.walk(CSRC):
        hs += [os.path.join(dirpath, f) for f in files if f.endswith((".h", ".cuh"))]
    return hs


def _compile(nvcc, src, obj):
    cmd = [nvcc] + ARCH + COMMON + ["-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [nvcc, "-x", "cu"] + ARCH + COMMON + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose: bool = False, force: bool = False) -> str:
    nvcc = _nvcc()
    os.makedirs(OBJDIR, exist_ok=True)
    newest_header = max(os.path.getmtime(h) for h in _headers() if os.path.exists(h))
    jobs = []
    objs = []
    for src in _sources():
        rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
        obj = os.path.join(OBJDIR, rel + ".o")
        objs.append(obj)
        stale = (force or not os.path.exists(obj)
                 or os.path.getmtime(obj) < max(os.path.getmtime(src), newest_header))
        if stale:
            jobs.append((src, obj))
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            futs = [ex.submit(_compile, nvcc, s, o) for s, o in jobs]
            for f in futs:
                o = f.result()
                if verbose:
                    print("compiled", os.path.relpath(o, ROOT))
    if jobs or not os.path.exists(OUT):
        tmp = OUT + ".tmp"
        cmd = [nvcc] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs + ["-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, OUT)
        if verbose:
            print("linked", os.path.relpath(OUT, ROOT))
    _build_pyext(verbose, force)
    _build_examples(nvcc, verbose, force)
    return OUT


def _build_examples(nvcc, verbose: bool, force: bool) -> None:
    """User-op examples (examples/*.cu): each its own shared library, loaded
    with ctypes and registered through sfx_register_op (ops.register)."""
    exdir = os.path.join(PKG, "examples")
    if not os.path.isdir(exdir):
        return
    hdr = os.path.getmtime(os.path.join(ROOT, "include", "sfx.h"))
    for f in sorted(os.listdir(exdir)):
        if not f.endswith(".cu"):
            continue
        src = os.path.join(exdir, f)
        out = os.path.join(PKG, "libsfx_" + f[:-3] + ".so")
        if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(src), hdr):
            continue
        cmd = [nvcc] + ARCH + COMMON + ["-shared", "-cudart", "static", src, "-o", out + ".tmp"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"example build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(out + ".tmp", out)
        if verbose:
            print("linked", os.path.relpath(out, ROOT))


def _build_pyext(verbose: bool, force: bool) -> None:
    """The optional CPython fast path for single-task submits (csrc/pyext/sfxfast.c),
    linked against libsfx.so (rpath $ORIGIN).  Failure is not fatal: the ctypes
    path stays in use."""
    import sysconfig

    src = os.path.join(CSRC, "pyext", "sfxfast.c")
    out = os.path.join(PKG, "_sfxfast" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))
    if not os.path.exists(src):
        return
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(src), os.path.getmtime(OUT)):
        return
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        return
    cmd = [cc, "-O2", "-shared", "-fPIC", "-I", sysconfig.get_paths()["include"], "-I", os.path.join(ROOT, "include"),
           src, "-o", out + ".tmp", "-L", PKG, "-l:libsfx.so", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        if verbose:
            print("python fast path not built:", r.stderr.strip()[:300])
        return
    os.replace(out + ".tmp", out)
    if verbose:
        print("linked", os.path.relpath(out, ROOT))


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
