#!/usr/bin/env python
"""Phase stamps of the dataflow POTRF's chain CTA (potrf_flow.cu built with
-DSFX_FLOW_PROF into a standalone binary).

    python tools/potrf_flow_probe.py            # builds tools/bin/flow_prof (nvcc, sm_100a)
    ./tools/bin/flow_prof [n] [mode]              # on the GPU box

Per step k: F = factor+invert 64x64 in registers, store = L/X stores + fdone,
Pw = wait for cnt[k+1][k], P = panel block product + store, Uw = wait for
cnt[k+1][k+1], Ul = load A_{k+1,k+1}, U = its update (registers).
"""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2308_15964_b200", "csrc", "kernels", "potrf_flow.cu")

MAIN = r'''
namespace sfx { std::atomic<unsigned long long> g_kernel_launches{0}; }
// F alone on one CTA: factor_inv64 on a 64x64 SPD block, timed with clock64
namespace sfx { namespace {
__global__ void __launch_bounds__(THREADS, 1) f_only_kernel(const double* A, long long* cyc, double* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const Patch pt = my_patch();
  load_block(s.c, A, 64);
  double a0[4][4], a[4][4], x[4][4];
  if (pt.lower) patch_load(a0, s.c, pt);
  long long best = 1ll << 60;
  for (int rep = 0; rep < 5; ++rep) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) a[r][c] = a0[r][c];
    __syncthreads();
    const long long t0 = clock64();
    factor_inv64(s, a, x, pt);
    __syncthreads();
    const long long t1 = clock64();
    if (t1 - t0 < best) best = t1 - t0;
  }
  if (threadIdx.x == 0) cyc[0] = best;
  double acc = 0;
  for (int r = 0; r < 4; ++r) for (int c = 0; c < 4; ++c) acc += a[r][c] + x[r][c];
  out[threadIdx.x] = acc;
}
} }
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1024;
  const int mode = argc > 2 ? atoi(argv[2]) : 2;
  std::vector<double> h(n * (size_t)n);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) h[i * (size_t)n + j] = (i == j ? n : 0.0) + 1.0 / (1 + std::abs(i - j));
  double* A; cudaMalloc(&A, h.size() * 8);
  const size_t wsb = 64 << 20;
  void* ws; cudaMalloc(&ws, wsb); cudaMemset(ws, 0, wsb);
  int* info; cudaMalloc(&info, 4); cudaMemset(info, 0, 4);
  for (int rep = 0; rep < 4; ++rep) {
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = sfx::launch_dpotrf_flow(A, n, n, info, ws, wsb, 0, mode);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("rep %d rc %d (%s): %.1f us\n", rep, (int)e, cudaGetErrorString(cudaGetLastError()), ms * 1e3);
  }
  {
    long long* cyc; double* out; cudaMallocManaged(&cyc, 64); cudaMalloc(&out, 4096 * 8);
    cudaFuncSetAttribute(sfx::f_only_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sfx::SMEM);
    sfx::f_only_kernel<<<1, 256, sfx::SMEM>>>(A, cyc, out);  // A now holds L: use the original
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    double* A64; cudaMalloc(&A64, 64 * 64 * 8);
    cudaMemcpy2D(A64, 64 * 8, A, n * 8, 64 * 8, 64, cudaMemcpyDeviceToDevice);
    sfx::f_only_kernel<<<1, 256, sfx::SMEM>>>(A64, cyc, out);
    cudaDeviceSynchronize();
    printf("F alone: %lld cycles (%.1f per pivot) %s\n", cyc[0], cyc[0] / 64.0, cudaGetErrorString(cudaGetLastError()));
  }
  unsigned long long p[64][8];
  cudaMemcpyFromSymbol(p, sfx::g_flow_prof, sizeof p);
  const int nb = n / 64;
  double tot[8] = {};
  for (int k = 0; k < nb; ++k) {
    double F = (p[k][1] - p[k][0]) / 1e3, st = (p[k][2] - p[k][1]) / 1e3;
    if (k + 1 == nb) { printf("k %2d: F %.1f store %.1f\n", k, F, st); break; }
    double Pw = (p[k][3] - p[k][2]) / 1e3, P = (p[k][4] - p[k][3]) / 1e3, Uw = (p[k][5] - p[k][4]) / 1e3,
           Ul = (p[k][6] - p[k][5]) / 1e3, U = (p[k][7] - p[k][6]) / 1e3, step = (p[k + 1][0] - p[k][0]) / 1e3;
    printf("k %2d: F %.1f store %.1f Pw %.1f P %.1f Uw %.1f Ul %.1f U %.1f | step %.1f\n", k, F, st, Pw, P, Uw, Ul, U, step);
  }
  printf("chain end -> kernel end not stamped; first F start to last F end: %.1f us\n", (p[nb - 1][2] - p[0][0]) / 1e3);
  return 0;
}
'''


VARIANTS = {
    "norest": [("""      double lr[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) lr[r] = crv[r] * r2;""", """      continue;
      double lr[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) lr[r] = crv[r] * r2;""")],
    "barsonly": [("""      const double d = s.col[buf][j];""", """      continue;
      const double d = s.col[buf][j];""")],
    # timing experiments only (wrong results): which part of the pivot loop costs what
}


def main():
    import sys
    variant = sys.argv[1] if len(sys.argv) > 1 else ""
    src = open(SRC).read()
    for old, new in VARIANTS.get(variant, []):
        assert old in src, old
        src = src.replace(old, new)
    os.makedirs(os.path.join(ROOT, "scratch"), exist_ok=True)
    out_src = os.path.join(ROOT, "scratch", f"flow_prof{variant}.cu")
    open(out_src, "w").write(src + MAIN)
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo", "-DSFX_FLOW_PROF",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "paper_2308_15964_b200", "csrc", "kernels"),
           out_src, "-o", os.path.join(ROOT, "tools", "bin", "flow_prof" + variant)]
    os.makedirs(os.path.join(ROOT, "tools", "bin"), exist_ok=True)
    subprocess.run(cmd, check=True)
    print("built tools/bin/flow_prof" + variant)


if __name__ == "__main__":
    main()
