#!/usr/bin/env python
"""Finer POTRF probe: timestamps inside factor64 (the 64x64 factor-and-invert).

    python tools/potrf_factor_probe.py     # builds scratch/fc_prof2 (nvcc, sm_100a)
    ./scratch/fc_prof2                     # on the GPU box

Extends tools/potrf_phase_probe.py's instrumented copy with globaltimer stamps
around each 16x16 warp Cholesky+inverse, panel, trailing update and the 64x64
inverse assembly (CTA 0, last factor_block call).
"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.chdir(ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
os.makedirs("scratch", exist_ok=True)
import potrf_phase_probe as pp
src = open(pp.SRC).read()
src = pp.instrument(src)
src = src.replace("__device__ unsigned long long g_prof[16][8];",
                  "__device__ unsigned long long g_prof[16][8];\n__device__ unsigned long long g_f[16];")
def stamp(slot):
    return f"if (blockIdx.x == 0 && threadIdx.x == 0) g_f[{slot}] = gt();"
pairs = [
 ("  for (int p = 0; p < 4; ++p) {\n    const int o = 16 * p;\n    if (warp == 0) warp_potrf_inv16(s.c, o, s.dinv[p], &s.bad);\n    __syncthreads();\n    if (p == 3) break;",
  "  for (int p = 0; p < 4; ++p) {\n    const int o = 16 * p;\n    " + "if (blockIdx.x == 0 && threadIdx.x == 0) g_f[4*p] = gt();" + "\n    if (warp == 0) warp_potrf_inv16(s.c, o, s.dinv[p], &s.bad);\n    __syncthreads();\n    if (blockIdx.x == 0 && threadIdx.x == 0) g_f[4*p+1] = gt();\n    if (p == 3) break;"),
 ("    // trailing lower update:", "    if (blockIdx.x == 0 && threadIdx.x == 0) g_f[4*p+2] = gt();\n    // trailing lower update:"),
 ("  const bool ok = s.bad == 0;\n  assemble_inv64(s);\n  return ok;",
  "  const bool ok = s.bad == 0;\n  " + stamp(13) + "\n  assemble_inv64(s);\n  " + stamp(14) + "\n  return ok;"),
]
for o, n in pairs:
    assert o in src, o[:50]
    src = src.replace(o, n)
# print g_f after the run: piggyback on main's printf of factor0
src = src.replace('printf("factor0', 'unsigned long long f[16]; cudaMemcpyFromSymbol(f, g_f, sizeof(f)); '
                  'for (int q = 0; q < 4; ++q) printf("p%d potrf16 %.2f panel %.2f trailing %.2f\\n", q, (f[4*q+1]-f[4*q])/1e3, q<3?(f[4*q+2]-f[4*q+1])/1e3:0.0, q<3?(f[4*q+4]-f[4*q+2])/1e3:0.0); printf("assemble %.2f total %.2f\\n", (f[14]-f[13])/1e3, (f[14]-f[0])/1e3); printf("factor0')
open("scratch/fc_prof2.cu", "w").write(src)

kern = "paper_2308_15964_b200/csrc"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-I", "include", "-I", kern,
                "-I", kern + "/kernels", "-o", "scratch/fc_prof2", "scratch/fc_prof2.cu"], check=True)
print("built")
