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

// X L^T = B for a leaf of <= 64 columns (L padded with identity to 64).
// One thread per row of B: the row lives in registers and is solved
// right-looking (x_j = b_j / L_jj, then b_i -= L_ij x_j for every i > j), so
// each step is a run of independent FMAs instead of a dependent dot product.
// B rows are staged through shared memory so global loads/stores coalesce.
__global__ void __launch_bounds__(LEAF) trsm_leaf_kernel(double* B, long long ldb, int M, int n, const double* L,
                                                         long long ldl) {
  // one buffer, used as the B staging area and then as LsT[j][i] = L[i][j]
  __shared__ double buf[LEAF][LEAF + 1];
  const int tid = threadIdx.x;
  const int r0 = blockIdx.x * LEAF;
#pragma unroll 16
  for (int e = tid; e < LEAF * LEAF; e += LEAF) {
    const int i = e / LEAF, j = e % LEAF;  // coalesced over j
    const int r = r0 + i;
    buf[i][j] = (r < M && j < n) ? B[r * ldb + j] : 0.0;
  }
  __syncthreads();
  double x[LEAF];
#pragma unroll
  for (int c = 0; c < LEAF; ++c) x[c] = buf[tid][c];
  __syncthreads();
#pragma unroll 16
  for (int e = tid; e < LEAF * LEAF; e += LEAF) {
    const int i = e / LEAF, j = e % LEAF;
    double v = (i == j) ? 1.0 : 0.0;
    if (i < n && j < n && j <= i) v = L[i * ldl + j];
    buf[j][i] = v;
  }
  __syncthreads();
  double(*LsT)[LEAF + 1] = buf;
#pragma unroll
  for (int j = 0; j < LEAF; ++j) {
    x[j] = x[j] / LsT[j][j];
#pragma unroll
    for (int i = j + 1; i < LEAF; ++i) x[i] = fma(-LsT[j][i], x[j], x[i]);
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < LEAF; ++c) buf[tid][c] = x[c];
  __syncthreads();
#pragma unroll 16
  for (int e = tid; e < LEAF * LEAF; e += LEAF) {
    const int i = e / LEAF, j = e % LEAF;
    const int r = r0 + i;
    if (r < M && j < n) B[r * ldb + j] = buf[i][j];
  }
}

// In-place lower Cholesky of a <= 64 leaf (padded with identity): 256 threads,
// each owning a 4x4 block of the lower triangle in registers (outer-product
// form, column scaling deferred).  Column j is broadcast through a
// double-buffered shared vector: one barrier and <= 16 FMAs per thread per step.
__global__ void __launch_bounds__(256) potrf_leaf_kernel(double* A, long long lda, int n, int* info, int off) {
  __shared__ double colbuf[2][LEAF];
  __shared__ double pivs[LEAF];
  __shared__ int first_bad;
  if (threadIdx.x == 0) first_bad = LEAF + 1;
  const int tid = threadIdx.x;
  const int ti = tid >> 4, tk = tid & 15;
  const int R = ti * 4, C = tk * 4;
  const bool active = tk <= ti;
  double a[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = R + r, k = C + c;
      double v = (i == k) ? 1.0 : 0.0;
      if (active && i < n && k < n && k <= i) v = A[i * lda + k];
      a[r][c] = v;
    }
  for (int j = 0; j < LEAF; ++j) {
    const int buf = j & 1;
    if (active && tk == (j >> 2)) {
      const int jj = j & 3;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const double v = jj == 0 ? a[r][0] : jj == 1 ? a[r][1] : jj == 2 ? a[r][2] : a[r][3];
        colbuf[buf][R + r] = v;
      }
    }
    __syncthreads();
    const double piv = colbuf[buf][j];
    if (tid == 0) pivs[j] = piv;
    if (active && C + 3 > j) {
      const double inv = 1.0 / piv;
      double cr[4], cc[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) cr[r] = colbuf[buf][R + r] * inv;
#pragma unroll
      for (int c = 0; c < 4; ++c) cc[c] = colbuf[buf][C + c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (C + c > j && R + r >= C + c) a[r][c] = fma(-cr[r], cc[c], a[r][c]);
    }
  }
  __syncthreads();
  if (tid < LEAF && tid < n && !(pivs[tid] > 0.0)) atomicMin(&first_bad, tid + 1);
  __syncthreads();
  // info (mapped host word): leaves run in column order on one stream, so the first
  // failing leaf stores first; LAPACK info = order of the first non-positive minor
  if (tid == 0 && info && first_bad <= LEAF && *reinterpret_cast<volatile int*>(info) == 0)
    *reinterpret_cast<volatile int*>(info) = off + first_bad;
  if (!active) return;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = R + r, k = C + c;
      if (i < n && k < n && k <= i) A[i * lda + k] = (i == k) ? sqrt(pivs[i]) : a[r][c] / sqrt(pivs[k]);
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
    count_launch();
    trsm_leaf_kernel<<<(M + LEAF - 1) / LEAF, LEAF, 0, s>>>(B, ldb, M, n, L, ldl);
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

cudaError_t launch_dpotrf(double* A, long long lda, int n, int* info, cudaStream_t s, int off) {
  if (n <= 0) return cudaSuccess;
  if (n <= LEAF) {
    count_launch();
    potrf_leaf_kernel<<<1, 256, 0, s>>>(A, lda, n, info, off);
    return cudaGetLastError();
  }
  const int n1 = split(n), n2 = n - n1;
  cudaError_t e = launch_dpotrf(A, lda, n1, info, s, off);
  if (e) return e;
  // A21 <- A21 * L11^-T
  e = launch_dtrsm(A, lda, A + n1 * lda, lda, n2, n1, s);
  if (e) return e;
  // A22 -= A21 A21^T (lower)
  e = launch_dgemm(A + n1 * lda, lda, A + n1 * lda, lda, A + n1 * lda + n1, lda, n2, n2, n1, -1.0, 1.0, true, true, s);
  if (e) return e;
  return launch_dpotrf(A + n1 * lda + n1, lda, n2, info, s, off + n1);
}

}  // namespace sfx
