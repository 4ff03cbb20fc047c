#!/usr/bin/env python
"""Build and run an instrumented copy of the cooperative POTRF (phase timestamps).

    python tools/potrf_phase_probe.py            # builds scratch/fc_prof (nvcc, sm_100a)
    ./scratch/fc_prof                            # on the GPU box

The copy adds globaltimer stamps on CTA 0 around every phase of every 64-wide
block step of potrf_coop_kernel and a main() that factors one 1024 x 1024 SPD
matrix; output: per-step panel / barrier / next-diagonal update / factor_block
times (profiles/r1d_potrf_phases.md).
"""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2308_15964_b200", "csrc", "kernels", "factor_coop.cu")


def instrument(src: str) -> str:
    src = src.replace('#include "kernels.h"', '#include "kernels.h"\n'
                      '__device__ unsigned long long g_prof[16][8];\n'
                      '__device__ __forceinline__ unsigned long long gt(){unsigned long long t; '
                      'asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;}\n'
                      '#define PROF(kb, slot) do { if (blockIdx.x == 0 && threadIdx.x == 0 && (kb) < 16) '
                      'g_prof[(kb)][(slot)] = gt(); } while (0)')
    pairs = [
        ("  if (blockIdx.x == 0) factor_block(s, A, lda, 0, ws, info, store_inv);\n  grid_barrier(bar);\n",
         "  PROF(0, 0);\n  if (blockIdx.x == 0) factor_block(s, A, lda, 0, ws, info, store_inv);\n  PROF(0, 1);\n"
         "  grid_barrier(bar);\n  PROF(0, 2);\n"),
        ("      store_tile(Aik, lda, acc, false, nullptr);\n    }\n    grid_barrier(bar);",
         "      store_tile(Aik, lda, acc, false, nullptr);\n    }\n    PROF(kb, 3);\n    grid_barrier(bar);\n"
         "    PROF(kb, 4);"),
        ("        factor_block(s, A, lda, kb + 1, ws, info, store_inv);\n      }\n    }\n    grid_barrier(bar);",
         "        PROF(kb, 5);\n        factor_block(s, A, lda, kb + 1, ws, info, store_inv);\n        PROF(kb, 6);\n"
         "      }\n    }\n    grid_barrier(bar);\n    PROF(kb, 7);"),
    ]
    for old, new in pairs:
        assert old in src, old[:60]
        src = src.replace(old, new)
    return src + MAIN


MAIN = r'''
namespace sfx { std::atomic<unsigned long long> g_kernel_launches{0};
cudaError_t launch_dgemm_group(const GemmDesc*, int, int, int, int, double, double, bool, bool, cudaStream_t, bool) {
  return cudaErrorNotSupported; } }
#include <cstdio>
#include <vector>
#include <cmath>
int main() {
  const int n = 1024;
  std::vector<double> h(n * (size_t)n);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) h[i * (size_t)n + j] = (i == j ? n : 0.0) + 1.0 / (1 + std::abs(i - j));
  double* A; cudaMalloc(&A, h.size() * 8);
  void* ws; cudaMalloc(&ws, 64 << 20); cudaMemset(ws, 0, 64 << 20);
  int* info; cudaMalloc(&info, 4);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = sfx::launch_dpotrf_coop(A, n, n, info, ws, 0, true);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("rep %d rc %d: %.1f us\n", rep, (int)e, ms * 1e3);
  }
  unsigned long long p[16][8];
  cudaMemcpyFromSymbol(p, g_prof, sizeof p);
  printf("factor0 %.1f us, barrier0 %.1f\n", (p[0][1] - p[0][0]) / 1e3, (p[0][2] - p[0][1]) / 1e3);
  for (int kb = 0; kb < 15; ++kb) {
    unsigned long long s = kb == 0 ? p[0][2] : p[kb - 1][7];
    printf("kb %2d: panel %.1f  bar1 %.1f  next-diag update %.1f  factor %.1f  rest+bar2 %.1f  | step %.1f\n", kb,
           (p[kb][3] - s) / 1e3, (p[kb][4] - p[kb][3]) / 1e3, (p[kb][5] - p[kb][4]) / 1e3, (p[kb][6] - p[kb][5]) / 1e3,
           (p[kb][7] - p[kb][6]) / 1e3, (p[kb][7] - s) / 1e3);
  }
  return 0;
}
'''


def main():
    os.makedirs(os.path.join(ROOT, "scratch"), exist_ok=True)
    out = os.path.join(ROOT, "scratch", "fc_prof.cu")
    with open(out, "w") as fh:
        fh.write(instrument(open(SRC).read()))
    kern = os.path.join(ROOT, "paper_2308_15964_b200", "csrc")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "-I", os.path.join(ROOT, "include"), "-I", kern, "-I", os.path.join(kern, "kernels"),
                    "-o", os.path.join(ROOT, "scratch", "fc_prof"), out], check=True)
    print("built scratch/fc_prof")


if __name__ == "__main__":
    main()
