// Full triangular inverse for the Cholesky critical path (POTRF -> TRSM).
//
// DPOTRF with store_inverses = 2 ("full"): after the cooperative blocked
// factorization (which leaves inv(L_jj)^T of every 64x64 diagonal block in that
// block's strict upper triangle), the inverse W = inv(L) of the whole b x b
// factor is built by recursive doubling on the DMMA GEMM kernel:
//
//     inv([[L11, 0], [L21, L22]]) = [[W11, 0], [-W22 L21 W11, W22]]
//
// level s = 64, 128, ..., b/2: for every pair of s-blocks on the diagonal,
// T = L21 W11 then W21 = -W22 T (two grouped DGEMM launches per level, all pairs
// of a level in one launch).  W is kept dense (zero upper triangle) in the
// stream's scratch; at the end W^T's strict upper triangle is written to the
// tile's strict upper triangle (the factor L in the lower triangle is
// untouched, LAPACK 'L' semantics for the part the oracle compares).
//
// DTRSM with inverse = 2: X = B L^-T = B W^T is then ONE NN DGEMM whose B
// operand is the tile's upper triangle read with the TRI mask (k > n -> 0,
// k == n -> 1 / L_nn), k-tiles below the diagonal skipped, into scratch and
// copied back: fully parallel, instead of 16 dependent block-column sweeps.
//
// Accuracy: multiplying by an explicit triangular inverse has an error bound
// growing with cond(L) (vs cond(L_jj) of 64x64 blocks for the block-inverse
// sweeps); for the SPD tiles of the tiled Cholesky this is far inside the
// stated tolerances (tests/test_gpu_ops.py).
#include "kernels.h"

namespace sfx {
namespace {

// W (dense n x n, zero-initialised) <- the inverses of the 64x64 diagonal blocks:
// W[i][j] = 1 / A[i][i] (i == j), A[j][i] (i > j, same block: the stored inv^T)
__global__ void expand_diag_inv_kernel(const double* A, long long lda, double* W, int n) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;  // over the 64x64 blocks' elements
  const int nb = n / 64;
  if (e >= nb * 64 * 64) return;
  const int blk = e >> 12, r = (e >> 6) & 63, c = e & 63;
  const int i = blk * 64 + r, j = blk * 64 + c;
  double v = 0.0;
  if (r == c)
    v = 1.0 / A[static_cast<long long>(i) * lda + i];
  else if (r > c)
    v = A[static_cast<long long>(j) * lda + i];
  W[static_cast<long long>(i) * n + j] = v;
}

// A[p][q] = W[q][p] for p < q (strict upper triangle), 32x32 smem-tiled transpose
__global__ void store_upper_transposed_kernel(double* A, long long lda, const double* W, int n) {
  __shared__ double t[32][33];
  const int bq = blockIdx.x, bp = blockIdx.y;  // output tile: rows p in bp*32.., cols q in bq*32..
  if (bq < bp) return;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int k = ty; k < 32; k += 8) t[k][tx] = W[static_cast<long long>(bq * 32 + k) * n + bp * 32 + tx];
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int p = bp * 32 + k, q = bq * 32 + tx;
    if (p < q) A[static_cast<long long>(p) * lda + q] = t[tx][k];
  }
}

}  // namespace

bool fullinv_supported(int n) {
  if (n < 128 || n > 2048 || n % 64) return false;
  const int nb = n / 64;
  return (nb & (nb - 1)) == 0;  // power-of-two number of 64-blocks: exact doubling
}

// [coop POTRF workspace (barrier + block inverses)] [W: n x n] [T: n x n / 4]
static size_t w_offset(int n) { return (coop_workspace_bytes(n) + (1ull << 20) - 1) >> 20 << 20; }

size_t fullinv_workspace_bytes(int n) {
  return w_offset(n) + static_cast<size_t>(n) * n * 8 + static_cast<size_t>(n) * n / 4 * 8;
}

cudaError_t launch_dpotrf_fullinv(double* A, long long lda, int n, int* info, void* workspace, size_t ws_bytes,
                                  cudaStream_t s) {
  if (!fullinv_supported(n) || ws_bytes < fullinv_workspace_bytes(n)) return cudaErrorInvalidValue;
  cudaError_t e = launch_dpotrf_coop(A, lda, n, info, workspace, s, true);
  if (e != cudaSuccess) return e;
  double* W = reinterpret_cast<double*>(static_cast<char*>(workspace) + w_offset(n));
  double* T = W + static_cast<size_t>(n) * n;
  e = cudaMemsetAsync(W, 0, static_cast<size_t>(n) * n * 8, s);
  if (e != cudaSuccess) return e;
  const int nelem = (n / 64) * 64 * 64;
  count_launch();
  expand_diag_inv_kernel<<<(nelem + 255) / 256, 256, 0, s>>>(A, lda, W, n);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  GemmDesc d1[32], d2[32];
  for (int sz = 64; 2 * sz <= n; sz *= 2) {
    const int pairs = n / (2 * sz);
    e = cudaMemsetAsync(T, 0, static_cast<size_t>(pairs) * sz * sz * 8, s);
    if (e != cudaSuccess) return e;
    for (int p = 0; p < pairs; ++p) {
      const long long o = static_cast<long long>(p) * 2 * sz;
      double* Tp = T + static_cast<size_t>(p) * sz * sz;
      // T = L21 W11   (L21: rows o+sz.., cols o.. of the factor; W11 at (o, o))
      d1[p] = GemmDesc{A + (o + sz) * lda + o, lda, W + o * n + o, n, Tp, sz};
      // W21 = -W22 T  (W22 at (o+sz, o+sz); W21 at (o+sz, o), zero before)
      d2[p] = GemmDesc{W + (o + sz) * n + (o + sz), n, Tp, sz, W + (o + sz) * n + o, n};
    }
    // ldc differs between T (sz) and W (n): separate launches per level.  A single
    // cooperative launch of the levels with 64^3 DFMA block products was slower
    // (1182 vs 1097 us for b = 1024): the DMMA kernel with split-K wins.
    if ((e = launch_dgemm_group(d1, pairs, sz, sz, sz, 1.0, 1.0, false, false, s)) != cudaSuccess) return e;
    if ((e = launch_dgemm_group(d2, pairs, sz, sz, sz, -1.0, 1.0, false, false, s)) != cudaSuccess) return e;
  }
  count_launch();
  dim3 grid(n / 32, n / 32), block(32, 8);
  store_upper_transposed_kernel<<<grid, block, 0, s>>>(A, lda, W, n);
  return cudaGetLastError();
}

cudaError_t launch_dtrsm_fullinv(const double* L, long long ldl, double* B, long long ldb, int M, int n, void* scratch,
                                 size_t bytes, cudaStream_t s) {
  const size_t need = static_cast<size_t>(M) * n * 8;
  if (!scratch || bytes < need) return cudaErrorInvalidValue;
  double* X = static_cast<double*>(scratch);
  cudaError_t e = cudaMemsetAsync(X, 0, need, s);
  if (e != cudaSuccess) return e;
  GemmDesc d{B, ldb, L, ldl, X, n};
  // X = B U, U = upper triangle of the tile with reciprocal diagonal (TRI mask)
  if ((e = launch_dgemm_group(&d, 1, M, n, n, 1.0, 1.0, false, false, s, true)) != cudaSuccess) return e;
  return cudaMemcpy2DAsync(B, ldb * 8, X, static_cast<size_t>(n) * 8, static_cast<size_t>(n) * 8, M,
                           cudaMemcpyDeviceToDevice, s);
}

}  // namespace sfx
