// Tile DTRSM (B <- B * L^-T) and DPOTRF (A = L L^T, lower) for sm_100a.
//
// Both are recursive: split the tile in two halves, solve/factor the leading
// half, update the trailing half with the DMMA GEMM/SYRK kernel (dgemm.cu),
// recurse.  Leaves (<= 64 columns) run in shared memory.  Every launch goes to
// the task's stream, so one tile task is one ordered kernel sequence and the
// runtime's end event covers all of it.  >97% of the flops of a 1024 tile land
// in the DMMA GEMM.
//
// Oracle: oracle/bodies.py trsm_rltn / potrf_l (scipy solve_triangular and
// numpy cholesky); the reference itself has no tile bodies.
#include "kernels.h"

namespace sfx {
namespace {

constexpr int LEAF = 64;
constexpr int TRSM_THREADS = 128;

// X L^T = B for a leaf: one thread per row of B, n <= 64 columns.
// x_j = (b_j - sum_{k<j} L[j][k] x_k) / L[j][j]
__global__ void __launch_bounds__(TRSM_THREADS) trsm_leaf_kernel(double* B, long long ldb, int M, int n,
                                                                   const double* L, long long ldl) {
  extern __shared__ double trsm_smem[];
  double(*Ls)[LEAF + 1] = reinterpret_cast<double(*)[LEAF + 1]>(trsm_smem);
  double(*xs)[TRSM_THREADS] = reinterpret_cast<double(*)[TRSM_THREADS]>(trsm_smem + LEAF * (LEAF + 1));
  const int tid = threadIdx.x;
  for (int e = tid; e < n * n; e += TRSM_THREADS) {
    const int j = e / n, k = e % n;
    Ls[j][k] = (k <= j) ? L[j * ldl + k] : 0.0;
  }
  const int r = blockIdx.x * TRSM_THREADS + tid;
  if (r < M)
    for (int j = 0; j < n; ++j) xs[j][tid] = B[r * ldb + j];
  __syncthreads();
  if (r < M) {
    for (int j = 0; j < n; ++j) {
      double s0 = xs[j][tid], s1 = 0.0;
      int k = 0;
      for (; k + 1 < j; k += 2) {
        s0 = fma(-Ls[j][k], xs[k][tid], s0);
        s1 = fma(-Ls[j][k + 1], xs[k + 1][tid], s1);
      }
      if (k < j) s0 = fma(-Ls[j][k], xs[k][tid], s0);
      xs[j][tid] = (s0 + s1) / Ls[j][j];
    }
    for (int j = 0; j < n; ++j) B[r * ldb + j] = xs[j][tid];
  }
}

// In-place lower Cholesky of an n <= 64 leaf in shared memory (outer-product
// form; the column scaling is deferred so each step needs one barrier).
__global__ void __launch_bounds__(256) potrf_leaf_kernel(double* A, long long lda, int n, int* info) {
  __shared__ double As[LEAF][LEAF + 1];
  const int tid = threadIdx.x;
  for (int e = tid; e < n * n; e += 256) {
    const int i = e / n, k = e % n;
    As[i][k] = (k <= i) ? A[i * lda + k] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double piv = As[j][j];
    if (piv <= 0.0) {
      if (tid == 0 && info) atomicCAS(info, 0, j + 1);
      return;
    }
    const double inv = 1.0 / piv;
    // trailing update A[i][k] -= A[i][j] * A[k][j] / A[j][j], j < k <= i
    const int m = n - j - 1;
    const int cnt = m * (m + 1) / 2;
    for (int e = tid; e < cnt; e += 256) {
      // e -> (ii, kk) with 0 <= kk <= ii < m
      int ii = static_cast<int>((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
      while ((ii + 1) * (ii + 2) / 2 <= e) ++ii;
      while (ii * (ii + 1) / 2 > e) --ii;
      const int kk = e - ii * (ii + 1) / 2;
      const int i = j + 1 + ii, k = j + 1 + kk;
      As[i][k] = fma(-As[i][j] * inv, As[k][j], As[i][k]);
    }
    __syncthreads();
  }
  for (int e = tid; e < n * n; e += 256) {
    const int i = e / n, k = e % n;
    if (k <= i) A[i * lda + k] = (i == k) ? sqrt(As[i][i]) : As[i][k] / sqrt(As[k][k]);
  }
}

int split(int n) {
  // leading half rounded to a multiple of the leaf (keeps GEMM operands aligned)
  int n1 = (n / 2 + LEAF - 1) / LEAF * LEAF;
  return n1 >= n ? n - LEAF : n1;
}

}  // namespace

cudaError_t launch_dtrsm(const double* L, long long ldl, double* B, long long ldb, int M, int n, cudaStream_t s) {
  if (M <= 0 || n <= 0) return cudaSuccess;
  if (n <= LEAF) {
    constexpr int smem = (LEAF * (LEAF + 1) + LEAF * TRSM_THREADS) * 8;
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr[dev & 63]) {
      cudaError_t e = cudaFuncSetAttribute(trsm_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e) return e;
      attr[dev & 63] = true;
    }
    count_launch();
    trsm_leaf_kernel<<<(M + TRSM_THREADS - 1) / TRSM_THREADS, TRSM_THREADS, smem, s>>>(B, ldb, M, n, L, ldl);
    return cudaGetLastError();
  }
  const int n1 = split(n), n2 = n - n1;
  cudaError_t e = launch_dtrsm(L, ldl, B, ldb, M, n1, s);
  if (e) return e;
  // B2 -= X1 * L21^T   (L21 = L[n1:, :n1] stored [n2 x n1] -> trans_b)
  e = launch_dgemm(B, ldb, L + n1 * ldl, ldl, B + n1, ldb, M, n2, n1, -1.0, 1.0, true, false, s);
  if (e) return e;
  return launch_dtrsm(L + n1 * ldl + n1, ldl, B + n1, ldb, M, n2, s);
}

cudaError_t launch_dpotrf(double* A, long long lda, int n, int* info, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n <= LEAF) {
    count_launch();
    potrf_leaf_kernel<<<1, 256, 0, s>>>(A, lda, n, info);
    return cudaGetLastError();
  }
  const int n1 = split(n), n2 = n - n1;
  cudaError_t e = launch_dpotrf(A, lda, n1, info, s);
  if (e) return e;
  // A21 <- A21 * L11^-T
  e = launch_dtrsm(A, lda, A + n1 * lda, lda, n2, n1, s);
  if (e) return e;
  // A22 -= A21 A21^T (lower)
  e = launch_dgemm(A + n1 * lda, lda, A + n1 * lda, lda, A + n1 * lda + n1, lda, n2, n2, n1, -1.0, 1.0, true, true, s);
  if (e) return e;
  return launch_dpotrf(A + n1 * lda + n1, lda, n2, info, s);
}

}  // namespace sfx
