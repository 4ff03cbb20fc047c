// Single-launch (cooperative) tile DPOTRF and DTRSM for the Cholesky critical path.
//
// The recursive versions in factor.cu issue ~100 small dependent launches per
// 1024x1024 tile; on the critical path (POTRF(k) -> TRSM(k+1,k) -> SYRK ->
// POTRF(k+1)) the launch gaps and tiny grids dominate.  Here one cooperative
// launch walks the 64-wide block columns with grid-wide barriers:
//
//   DPOTRF  for kb: [CTA 0] factor A_kk in registers, invert L_kk (64x64)
//                   barrier; panel A_ik <- A_ik * inv(L_kk)^T (one CTA per block)
//                   barrier; trailing A_ij -= A_ik A_jk^T (lower part of diagonal blocks)
//                   barrier
//   DTRSM   inverses of all 64x64 diagonal blocks of L (one CTA each); barrier;
//           for kb: X_{:,kb} <- B_{:,kb} * inv(L_kk)^T; barrier;
//                   B_{:,j} -= X_{:,kb} L_{j,kb}^T for j > kb; barrier
//
// Multiplying by the inverse of a 64x64 diagonal block (instead of substituting)
// is the standard blocked-TRSM formulation; its error grows with cond(L_kk) of
// the small block only.  Block products are 64x64x64 DFMA register tiles (4x4
// per thread) from K-major shared memory (conflict-free LDS.128).
// Oracle: oracle/bodies.py potrf / trsm (LAPACK semantics: upper triangle of
// the POTRF tile untouched).
#include <cooperative_groups.h>

#include <vector>

#include "kernels.h"

namespace sfx {
namespace {

constexpr int T = 64;       // block size
constexpr int P = T + 2;    // shared pitch (doubles): 528 B, 16-byte aligned rows
constexpr int THREADS = 256;
constexpr int COOP_GRID = 64;
constexpr int SMEM = 3 * T * P * 8 + 2 * T * 8 + T * 8 + 4 * 16 * 17 * 8 + 16;

struct Smem {
  double a[T][P];  // K-major operand A (a[k][m])
  double b[T][P];  // K-major operand B (b[k][n])
  double c[T][P];  // scratch / row-major tile
  double col[2][T];
  double piv[T];
  double dinv[4][16][17];  // inverses of the four 16x16 diagonal sub-blocks
  int bad;
};

// Sense-free grid barrier: counter returns to 0, generation only grows.
__device__ void grid_barrier(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = bar + 1;
    const unsigned int g0 = *gen;
    __threadfence();
    const unsigned int arrived = atomicAdd(bar, 1u) + 1;
    if (arrived == gridDim.x) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g0) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

// dst[k][m] = src[m][k] (64x64 block, global row-major).  All 8 16-byte loads
// of a thread are issued before any shared store: one memory round trip per block.
__device__ __forceinline__ void load_T(double (*dst)[P], const double* src, long long ld) {
  double2 v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * THREADS;  // pair index: row m = e >> 5, cols 2*(e & 31)
    v[u] = *reinterpret_cast<const double2*>(src + (e >> 5) * ld + 2 * (e & 31));
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * THREADS;
    const int m = e >> 5, k = 2 * (e & 31);
    dst[k][m] = v[u].x;
    dst[k + 1][m] = v[u].y;
  }
}

// dst[r][c] = src[r][c]
__device__ __forceinline__ void load_N(double (*dst)[P], const double* src, long long ld) {
  double2 v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * THREADS;
    v[u] = *reinterpret_cast<const double2*>(src + (e >> 5) * ld + 2 * (e & 31));
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * THREADS;
    *reinterpret_cast<double2*>(&dst[e >> 5][2 * (e & 31)]) = v[u];
  }
}

// acc[r][c] += sum_k A[m][k] B[n][k] over the thread's 4x4 patch (m = 4ty+r, n = 4tx+c),
// operands K-major in shared memory
__device__ __forceinline__ void mm_nt(double acc[4][4], const double (*AT)[P], const double (*BT)[P]) {
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
#pragma unroll 4
  for (int k = 0; k < T; ++k) {
    const double2 a01 = *reinterpret_cast<const double2*>(&AT[k][4 * ty]);
    const double2 a23 = *reinterpret_cast<const double2*>(&AT[k][4 * ty + 2]);
    const double2 b01 = *reinterpret_cast<const double2*>(&BT[k][4 * tx]);
    const double2 b23 = *reinterpret_cast<const double2*>(&BT[k][4 * tx + 2]);
    const double av[4] = {a01.x, a01.y, a23.x, a23.y};
    const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = fma(av[r], bv[c], acc[r][c]);
  }
}

// ---- blocked 64x64 Cholesky + inverse: 16-wide sub-blocks factored and inverted
//      by single warps (only __syncwarp), panel/trailing/inverse assembly by the
//      whole CTA: ~20 CTA barriers per 64 block instead of ~130 ----

// 1/sqrt(d) to ~1 ulp: MUFU approximation + two Newton steps (no slow-path
// branch, no IEEE division on the dependent chain)
__device__ __forceinline__ double rsqrt_refined(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double h = 0.5 * d;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

// warp: X = inv(L) column by column, right-looking: lane n holds column n of X
// in x[]; after x[q] is final every later row k gets acc_k -= L[k][q] x[q].  The
// dependent chain per step is one multiply + one fma (the shuffles of L[k][q]
// do not depend on x and issue early).  rinv[q] = 1 / L[q][q].
__device__ __forceinline__ void warp_trinv16(const double (&r)[16], const double (&rinv)[16], int n,
                                             double (&x)[16]) {
#pragma unroll
  for (int q = 0; q < 16; ++q) x[q] = (q == n) ? 1.0 : 0.0;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    x[q] *= rinv[q];  // rows q < n stay exactly 0
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      if (k > q) {
        const double lkq = __shfl_sync(0xffffffffu, r[q], k);  // L[k][q] from lane k
        x[k] = fma(-lkq, x[q], x[k]);
      }
    }
  }
}

// warp: in-place lower Cholesky of the 16x16 block c[o..o+16)^2 (Schur complement)
// and its inverse into x.  Lane i (< 16) keeps row i in registers; columns are
// broadcast with shuffles, so the 16 dependent steps need no shared-memory
// round trips.  Every lane computes every pivot's 1/sqrt, so the inverse needs
// no division at all.
__device__ __forceinline__ void warp_potrf_inv16(double (*c)[P], int o, double (*x)[17], int* bad) {
  const int lane = threadIdx.x & 31;
  const int i = lane & 15;
  double r[16], rinv[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) r[k] = (k <= i) ? c[o + i][o + k] : 0.0;
  int first_bad = 0;  // 1-based pivot index of the first non-positive pivot (warp-uniform)
#pragma unroll 16
  for (int j = 0; j < 16; ++j) {
    const double d = __shfl_sync(0xffffffffu, r[j], j);  // pivot (Schur complement) from lane j
    if (!(d > 0.0) && first_bad == 0) first_bad = j + 1;
    const double rs = rsqrt_refined(d);
    rinv[j] = rs;
    // scale column j below the diagonal, then the rank-1 update of the trailing rows.
    // selects, not `if (i == j) r[j] = ..`: equality propagation would turn that
    // into r[i] (a dynamic index) and push r[] to local memory
    const double rj = r[j];
    r[j] = (i > j) ? rj * rs : ((i == j) ? d * rs : rj);
    // fixed trip counts (k > j tested inside) so both loops unroll fully and
    // r[] stays in registers; the test is warp-uniform, the shuffle is safe
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      if (k > j) {
        const double lkj = __shfl_sync(0xffffffffu, r[j], k);  // L[k][j] from lane k
        if (i >= k) r[k] = fma(-r[j], lkj, r[k]);
      }
    }
  }
  if (first_bad && lane == 0 && *bad == 0) *bad = o + first_bad;  // 1-based column in the 64-block
  if (lane < 16) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k <= i) c[o + i][o + k] = r[k];
  }
  double xs[16];
  warp_trinv16(r, rinv, i, xs);
  if (lane < 16) {
#pragma unroll
    for (int q = 0; q < 16; ++q) x[q][i] = xs[q];
  }
  __syncwarp();
}

// warp: inverse of an already-factored lower 16x16 block (lane n: column n)
__device__ __forceinline__ void warp_inv16(const double (*c)[P], int o, double (*x)[17]) {
  const int lane = threadIdx.x & 31;
  const int i = lane & 15;
  double r[16], rinv[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) r[k] = (k <= i) ? c[o + i][o + k] : 0.0;
#pragma unroll
  for (int q = 0; q < 16; ++q) rinv[q] = 1.0 / __shfl_sync(0xffffffffu, r[q], q);  // independent: ILP
  double xs[16];
  warp_trinv16(r, rinv, i, xs);
  if (lane < 16) {
#pragma unroll
    for (int q = 0; q < 16; ++q) x[q][i] = xs[q];
  }
  __syncwarp();
}

// CTA: full inverse of the lower 64x64 L in s.c from the four 16x16 diagonal
// inverses in s.dinv: X_pq = -D_p^{-1} sum_{q<=r<p} L_pr X_rq, block row by
// block row.  Result: s.b[k][n] = inv(L)[n][k] (K-major operand for mm_nt);
// s.a is scratch (row-major X).
__device__ void assemble_inv64(Smem& s) {
  const int tid = threadIdx.x;
  for (int e = tid; e < T * T; e += THREADS) {
    const int i = e >> 6, n = e & 63;
    const int p = i >> 4, q = n >> 4;
    s.a[i][n] = (p == q) ? s.dinv[p][i & 15][n & 15] : 0.0;
  }
  __syncthreads();
  for (int p = 1; p < 4; ++p) {
    // T_pq = sum_{r=q}^{p-1} L_pr X_rq for every q < p (kept in registers, <= 3 per thread)
    double t[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) {  // static register indices (no local-memory array)
      const int e = tid + u * THREADS;
      t[u] = 0.0;
      if (e < p * 256) {
        const int q = e >> 8, ii = (e >> 4) & 15, nn = e & 15;
        const int i = 16 * p + ii, n = 16 * q + nn;
        double acc = 0.0;
        for (int k = 16 * q; k < 16 * p; ++k) acc = fma(s.c[i][k], s.a[k][n], acc);
        t[u] = acc;
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 3; ++u) {  // park T in the (still zero) X_pq slots
      const int e = tid + u * THREADS;
      if (e < p * 256) s.a[16 * p + ((e >> 4) & 15)][16 * (e >> 8) + (e & 15)] = t[u];
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 3; ++u) {  // X_pq = -D_p^{-1} T_pq
      const int e = tid + u * THREADS;
      if (e < p * 256) {
        const int q = e >> 8, ii = (e >> 4) & 15, nn = e & 15;
        double acc = 0.0;
        for (int k = 0; k <= ii; ++k) acc = fma(s.dinv[p][ii][k], s.a[16 * p + k][16 * q + nn], acc);
        t[u] = -acc;
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int e = tid + u * THREADS;
      if (e < p * 256) s.a[16 * p + ((e >> 4) & 15)][16 * (e >> 8) + (e & 15)] = t[u];
    }
    __syncthreads();
  }
  for (int e = tid; e < T * T; e += THREADS) {
    const int r = e >> 6, c = e & 63;
    s.b[r][c] = s.a[c][r];  // b[k][n] = inv[n][k]
  }
  __syncthreads();
}

// CTA: s.c (row-major, lower part = SPD block) <- L (upper zeroed); s.b <- inv(L)^T
// K-major.  Returns false if a pivot was not positive.
__device__ bool factor64(Smem& s) {
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) s.bad = 0;
  for (int e = tid; e < T * T; e += THREADS) {
    const int i = e >> 6, k = e & 63;
    if (k > i) s.c[i][k] = 0.0;
  }
  __syncthreads();
  for (int p = 0; p < 4; ++p) {
    const int o = 16 * p;
    if (warp == 0) warp_potrf_inv16(s.c, o, s.dinv[p], &s.bad);
    __syncthreads();
    if (p == 3) break;
    // panel rows below: c[r][o..o+16) <- c[r][o..o+16) * D_p^{-T}
    const int rows = T - o - 16;
    double v[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int e = tid + u * THREADS;
      v[u] = 0.0;
      if (e < rows * 16) {
        const int r = o + 16 + (e >> 4), q = e & 15;
        double acc = 0.0;
        for (int k = 0; k <= q; ++k) acc = fma(s.c[r][o + k], s.dinv[p][q][k], acc);
        v[u] = acc;
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int e = tid + u * THREADS;
      if (e < rows * 16) s.c[o + 16 + (e >> 4)][o + (e & 15)] = v[u];
    }
    __syncthreads();
    // trailing lower update: c[i][k] -= sum_q c[i][o+q] c[k][o+q], o+16 <= k <= i < 64;
    // threads walk the lower triangle only (row ii of it starts at ii(ii+1)/2)
    for (int e = tid; e < rows * (rows + 1) / 2; e += THREADS) {
      int ii = static_cast<int>((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
      while ((ii + 1) * (ii + 2) / 2 <= e) ++ii;
      while (ii * (ii + 1) / 2 > e) --ii;
      const int i = o + 16 + ii, k = o + 16 + (e - ii * (ii + 1) / 2);
      double acc = s.c[i][k];
#pragma unroll
      for (int q = 0; q < 16; ++q) acc = fma(-s.c[i][o + q], s.c[k][o + q], acc);
      s.c[i][k] = acc;
    }
    __syncthreads();
  }
  const bool ok = s.bad == 0;
  assemble_inv64(s);
  return ok;
}

// CTA: inverse of an already-factored lower 64x64 L in s.c (upper part ignored)
__device__ void inv64_blocked(Smem& s) {
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < T * T; e += THREADS) {
    const int i = e >> 6, k = e & 63;
    if (k > i) s.c[i][k] = 0.0;
  }
  __syncthreads();
  if (warp < 4) warp_inv16(s.c, 16 * warp, s.dinv[warp]);
  __syncthreads();
  assemble_inv64(s);
}

__device__ __forceinline__ void store_tile(double* dst, long long ld, const double acc[4][4], bool lower_only,
                                           const double (*orig)[P]) {
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int i = 4 * ty + r;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int k = 4 * tx + c;
      if (!lower_only || k <= i) dst[i * ld + k] = acc[r][c];
      else if (orig) dst[i * ld + k] = orig[i][k];
    }
  }
}

// factor the diagonal block kb in place (lower), inverse^T (K-major) to ws
__device__ void factor_block(Smem& s, double* A, long long lda, int kb, double* ws, int* info, int store_inv) {
  const int tid = threadIdx.x;
  double* Akk = A + (kb * T) * lda + kb * T;
  load_N(s.c, Akk, lda);
  __syncthreads();
  const bool ok = factor64(s);
  // info (mapped host word, see Backend::status_alloc): only CTA 0 factors diagonal
  // blocks, in order, so the first failing block is the first to store
  if (!ok && tid == 0 && info && *reinterpret_cast<volatile int*>(info) == 0)
    *reinterpret_cast<volatile int*>(info) = kb * T + s.bad;
  for (int e = tid; e < T * T; e += THREADS) {  // L back, original upper triangle kept
    const int i = e >> 6, k = e & 63;
    if (k <= i) Akk[i * lda + k] = s.c[i][k];
  }
  for (int e = tid; e < T * T; e += THREADS) {
    const int r = e >> 6, c = e & 63;
    ws[e] = s.b[r][c];
    if (store_inv && r < c) Akk[r * lda + c] = s.b[r][c];  // inv(L_kk)[c][r] in the strict upper triangle
  }
  __syncthreads();
}

__global__ void __launch_bounds__(THREADS) potrf_coop_kernel(double* A, long long lda, int nb, unsigned int* bar,
                                                              double* ws, int* info, int store_inv) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x;
  if (blockIdx.x == 0) factor_block(s, A, lda, 0, ws, info, store_inv);
  grid_barrier(bar);
  for (int kb = 0; kb + 1 < nb; ++kb) {
    // ---- panel: A_ik <- A_ik inv(L_kk)^T ----
    const int npanel = nb - 1 - kb;
    bool loaded = false;
    for (int w = blockIdx.x; w < npanel; w += gridDim.x) {
      if (!loaded) {
        for (int e = tid; e < T * T; e += THREADS) s.b[e >> 6][e & 63] = ws[e];
        loaded = true;
      }
      double* Aik = A + ((kb + 1 + w) * T) * lda + kb * T;
      load_T(s.a, Aik, lda);
      __syncthreads();
      double acc[4][4] = {};
      mm_nt(acc, s.a, s.b);
      __syncthreads();
      store_tile(Aik, lda, acc, false, nullptr);
    }
    grid_barrier(bar);
    // ---- trailing update A_ij -= A_ik A_jk^T, kb < j <= i; work item 0 is the
    //      next diagonal block: CTA 0 updates it first and factors it right away
    //      (overlapping the next POTRF step with this step's trailing update) ----
    const int ntiles = npanel * (npanel + 1) / 2;
    for (int w = blockIdx.x; w < ntiles; w += gridDim.x) {
      int ii = static_cast<int>((sqrtf(8.0f * w + 1.0f) - 1.0f) * 0.5f);
      while ((ii + 1) * (ii + 2) / 2 <= w) ++ii;
      while (ii * (ii + 1) / 2 > w) --ii;
      const int jj = w - ii * (ii + 1) / 2;
      const int ib = kb + 1 + ii, jb = kb + 1 + jj;
      double* Aij = A + (ib * T) * lda + jb * T;
      load_T(s.a, A + (ib * T) * lda + kb * T, lda);
      load_T(s.b, A + (jb * T) * lda + kb * T, lda);
      load_N(s.c, Aij, lda);
      __syncthreads();
      double acc[4][4];
      const int ty = tid >> 4, tx = tid & 15;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
      mm_nt(acc, s.a, s.b);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = s.c[4 * ty + r][4 * tx + c] - acc[r][c];
      __syncthreads();
      store_tile(Aij, lda, acc, ib == jb, nullptr);
      if (w == 0) {
        __syncthreads();
        factor_block(s, A, lda, kb + 1, ws, info, store_inv);
      }
    }
    grid_barrier(bar);
  }
}

struct TrsmTask {
  const double* L;
  double* B;
};

constexpr int TRSM_GROUP_MAX = 32;

struct TrsmGroup {
  TrsmTask t[TRSM_GROUP_MAX];
  int ntasks, mb, nb;
  long long ldl, ldb;
  unsigned int* bar;
  double* ws;  // ntasks * nb inverse blocks (64 x 64, K-major inverse transpose)
};

// One cooperative launch solves X L^T = B for every task of the group (shared
// barriers; work items are spread over the whole grid).
__global__ void __launch_bounds__(THREADS) trsm_coop_kernel(const __grid_constant__ TrsmGroup g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x;
  const int mb = g.mb, nb = g.nb;
  // ---- inverses of every diagonal block of every task's L ----
  for (int w = blockIdx.x; w < g.ntasks * nb; w += gridDim.x) {
    const int task = w / nb, j = w - task * nb;
    const double* Ljj = g.t[task].L + (j * T) * g.ldl + j * T;
    for (int e = tid; e < T * T; e += THREADS) {
      const int i = e >> 6, k = e & 63;
      s.c[i][k] = k <= i ? Ljj[i * g.ldl + k] : 0.0;
    }
    __syncthreads();
    inv64_blocked(s);
    double* out = g.ws + static_cast<long long>(w) * T * T;
    for (int e = tid; e < T * T; e += THREADS) out[e] = s.b[e >> 6][e & 63];
    __syncthreads();
  }
  grid_barrier(g.bar);
  for (int kb = 0; kb < nb; ++kb) {
    // ---- X_{:,kb} = B_{:,kb} inv(L_kk)^T ----
    for (int w = blockIdx.x; w < g.ntasks * mb; w += gridDim.x) {
      const int task = w / mb, rb = w - task * mb;
      const double* inv = g.ws + (static_cast<long long>(task) * nb + kb) * T * T;
      for (int e = tid; e < T * T; e += THREADS) s.b[e >> 6][e & 63] = inv[e];
      double* Bt = g.t[task].B + (rb * T) * g.ldb + kb * T;
      load_T(s.a, Bt, g.ldb);
      __syncthreads();
      double acc[4][4] = {};
      mm_nt(acc, s.a, s.b);
      __syncthreads();
      store_tile(Bt, g.ldb, acc, false, nullptr);
    }
    if (kb + 1 == nb) break;
    grid_barrier(g.bar);
    // ---- B_{:,j} -= X_{:,kb} L_{j,kb}^T, j > kb ----
    const int ncol = nb - 1 - kb;
    const int per_task = mb * ncol;
    for (int w = blockIdx.x; w < g.ntasks * per_task; w += gridDim.x) {
      const int task = w / per_task, t = w - task * per_task;
      const int rb = t / ncol, jb = kb + 1 + t % ncol;
      double* B = g.t[task].B;
      double* Bt = B + (rb * T) * g.ldb + jb * T;
      load_T(s.a, B + (rb * T) * g.ldb + kb * T, g.ldb);
      load_T(s.b, g.t[task].L + (jb * T) * g.ldl + kb * T, g.ldl);
      load_N(s.c, Bt, g.ldb);
      __syncthreads();
      double acc[4][4] = {};
      mm_nt(acc, s.a, s.b);
      const int ty = tid >> 4, tx = tid & 15;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = s.c[4 * ty + r][4 * tx + c] - acc[r][c];
      __syncthreads();
      store_tile(Bt, g.ldb, acc, false, nullptr);
    }
    grid_barrier(g.bar);
  }
}

int num_sms_coop() {
  static int n[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!n[dev & 63]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev & 63] = v > 0 ? v : 148;
  }
  return n[dev & 63];
}

bool set_smem_attrs() {
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (done[dev & 63]) return true;
  if (cudaFuncSetAttribute(potrf_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess)
    return false;
  if (cudaFuncSetAttribute(trsm_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess)
    return false;
  done[dev & 63] = true;
  return true;
}

}  // namespace

size_t coop_workspace_bytes(int n) { return 256 + static_cast<size_t>((n + T - 1) / T) * T * T * sizeof(double); }

bool coop_supported(int M, int n) { return n % T == 0 && M % T == 0 && n >= T && n <= 4096; }

cudaError_t launch_dpotrf_coop(double* A, long long lda, int n, int* info, void* workspace, cudaStream_t s,
                               bool store_inverses) {
  if (!set_smem_attrs()) return cudaErrorInvalidValue;
  unsigned int* bar = static_cast<unsigned int*>(workspace);
  double* ws = reinterpret_cast<double*>(static_cast<char*>(workspace) + 256);
  int nb = n / T;
  int store = store_inverses ? 1 : 0;
  void* args[] = {&A, &lda, &nb, &bar, &ws, &info, &store};
  count_launch();
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(potrf_coop_kernel), dim3(COOP_GRID), dim3(THREADS), args,
                                     SMEM, s);
}

cudaError_t launch_dtrsm_coop_group(const TrsmDesc* d, int ntasks, int M, int n, void* workspace, size_t ws_bytes,
                                    cudaStream_t s) {
  if (!set_smem_attrs()) return cudaErrorInvalidValue;
  const int mb = M / T, nb = n / T;
  for (int i0 = 0; i0 < ntasks; i0 += TRSM_GROUP_MAX) {
    const int cnt = ntasks - i0 < TRSM_GROUP_MAX ? ntasks - i0 : TRSM_GROUP_MAX;
    if (256 + static_cast<size_t>(cnt) * nb * T * T * sizeof(double) > ws_bytes) return cudaErrorMemoryAllocation;
    TrsmGroup g;
    for (int i = 0; i < cnt; ++i) {
      g.t[i].L = d[i0 + i].L;
      g.t[i].B = d[i0 + i].B;
      if (d[i0 + i].ldl != d[i0].ldl || d[i0 + i].ldb != d[i0].ldb) return cudaErrorInvalidValue;
    }
    g.ntasks = cnt;
    g.mb = mb;
    g.nb = nb;
    g.ldl = d[i0].ldl;
    g.ldb = d[i0].ldb;
    g.bar = static_cast<unsigned int*>(workspace);
    g.ws = reinterpret_cast<double*>(static_cast<char*>(workspace) + 256);
    // at most one CTA per SM: two concurrent cooperative grids always fit together
    int grid = cnt * mb * (nb > 1 ? nb - 1 : 1);
    if (grid > num_sms_coop()) grid = num_sms_coop();
    if (grid < 1) grid = 1;
    void* args[] = {&g};
    count_launch();
    cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(trsm_coop_kernel), dim3(grid), dim3(THREADS),
                                                args, SMEM, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_dtrsm_inv_group(const TrsmDesc* d, int ntasks, int M, int n, cudaStream_t s) {
  // Right-looking blocked TRSM on the DMMA GEMM kernel; the 64x64 diagonal
  // inverses come precomputed in L's upper triangle (store_inverses POTRF).
  const int nb = n / T;
  std::vector<GemmDesc> solve(ntasks), update(ntasks);
  for (int kb = 0; kb < nb; ++kb) {
    for (int i = 0; i < ntasks; ++i) {
      const double* Lkk = d[i].L + (kb * T) * d[i].ldl + kb * T;
      double* Bk = d[i].B + kb * T;
      // X_kb = B_kb * inv(L_kk)^T : NN with B-operand[k][n] = inv[n][k] = Lkk_upper[k][n]
      solve[i] = GemmDesc{Bk, d[i].ldb, Lkk, d[i].ldl, Bk, d[i].ldb};
    }
    cudaError_t e = launch_dgemm_group(solve.data(), ntasks, M, T, T, 1.0, 0.0, false, false, s, true);
    if (e != cudaSuccess) return e;
    const int rest = n - (kb + 1) * T;
    if (rest <= 0) break;
    for (int i = 0; i < ntasks; ++i) {
      const double* Ljk = d[i].L + ((kb + 1) * T) * d[i].ldl + kb * T;  // rows kb+1.. of column block kb
      update[i] = GemmDesc{d[i].B + kb * T, d[i].ldb, Ljk, d[i].ldl, d[i].B + (kb + 1) * T, d[i].ldb};
    }
    e = launch_dgemm_group(update.data(), ntasks, M, rest, T, -1.0, 1.0, true, false, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace sfx
