// Tile DPOTRF as ONE dataflow launch: 64x64 block tasks ordered by flags in
// global memory instead of grid-wide barriers, with the panel chain on one CTA.
//
// The cooperative kernel of factor_coop.cu walks the 64-wide block columns with
// three grid barriers per step and factors each 64x64 diagonal block with
// single-warp 16x16 steps: 48-59 us per step, 16 steps per 1024 tile, plus
// ~225 us of inverse doubling launches for the full-inverse TRSM
// (profiles/r1d_potrf_phases.md).  Here (b = 64 * nb):
//
//   chain (CTA 0), per step k:   F(k)  factor A_kk and invert it in registers
//                                      (one CTA barrier per pivot, below)
//                                P(k+1,k)   L_{k+1,k} = A_{k+1,k} X_kk^T
//                                U(k+1,k+1,k) A_{k+1,k+1} -= L L^T, kept on
//                                      chip -> F(k+1) starts at once
//   queue (CTAs 1.., ticketed):  P(i,k)   i >= k+2
//                                U(i,j,k) k+1 <= j <= i, (i,j) != (k+1,k+1),
//                                         rows in order (the chain's next
//                                         inputs come first)
//                                V(k+1,m) m <= k (store_inv == 2 only): block
//                                         X_{k+1,m} of the full inverse,
//                                         X_im = -X_ii sum_{q=m}^{i-1} L_iq X_qm
//
// Each block task waits (one thread spinning on an acquire load) for the flags
// of its inputs: fdone[k] (F), pdone[i][k] (P), cnt[i][j] = updates applied to
// A_ij (U, applied in k order, so the result is bitwise deterministic),
// vdone[i][k] (V).  Queue items are handed out in a topological order and the
// chain's inputs all come from earlier queue steps, so every wait terminates
// with all CTAs co-resident (cooperative launch).  A final grid barrier lets
// the CTAs clear the flags: the workspace is zero again for the next launch.
//
// Block products (64x64x64) run on the FP64 tensor path: mma.sync m8n8k4 ->
// DMMA.8x8x4, 8 warps x (32 x 16) warp tiles, operands row-major in shared
// memory with a 68-double pitch (conflict-free fragment loads), fed by
// cp.async (L2, never a stale L1 line of a block another CTA rewrote).  The
// first version's 4x4-per-thread DFMA products needed 4 shared bytes per FMA,
// twice what shared memory delivers at the FP64 rate (chain: P 7.5 us, U 5.7 us).
//
// F(k): thread (ty, tx) of 256 keeps the 4x4 patch rows 4ty.., columns 4tx.. of
// both the Schur complement a and of X~ (starts as I).  Pivot j: the owners of
// column j of a and row j of X~ publish them in shared memory (double
// buffered), ONE __syncthreads, then every thread computes 1/sqrt(a_jj) itself
// and applies  a_rc -= l_r l_c,  X~_rc -= l_r X_jc  (l = column j / sqrt(a_jj),
// zero for rows/columns <= j, which leaves the finished parts untouched); warps
// whose rows are all finished skip the updates.  The inverse rides along the
// factorization: X = inv(L) at the end.
//
// Outputs (LAPACK 'L' for the lower part): L in the lower triangle; store_inv
// 1: inv(L_kk)^T in the strict upper triangle of each 64x64 diagonal block
// (launch_dtrsm_inv_group), 2: inv(L)^T of the whole tile in its strict upper
// triangle (launch_dtrsm_fullinv's TRI-masked GEMM); 0: upper triangle untouched.
// Oracle: oracle/bodies.py potrf (numpy cholesky); tests/test_gpu_potrf_flow.py.
#include <cooperative_groups.h>

#include "kernels.h"

namespace sfx {
namespace {

// phase stamps of the chain CTA (tools/potrf_flow_probe.py builds with -DSFX_FLOW_PROF)
#ifdef SFX_FLOW_PROF
__device__ unsigned long long g_flow_prof[64][8];
__device__ __forceinline__ void prof(int k, int slot) {
  if (threadIdx.x == 0 && k < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_flow_prof[k][slot] = t;
  }
}
#else
__device__ __forceinline__ void prof(int, int) {}
#endif

constexpr int T = 64;
constexpr int PD = T + 4;  // shared pitch (doubles): 544 B rows, fragment loads conflict-free
constexpr int THREADS = 256;
constexpr int MAXNB = 64;  // n <= 4096

struct Smem {
  double a[T][PD];
  double b[T][PD];
  double c[T][PD];
  double d[T][PD];
  double col[2][T];
  double row[2][T];
  double rsv[T];  // F: 1/sqrt of each pivot (the deferred column / row scales)
  int off[MAXNB + 1];  // queue offsets per step
  int item;
  int bad;
  int pre;  // chain: operands of the next step prefetched during F
};
constexpr int SMEM = sizeof(Smem);

// flag area at the top of the workspace (zero between launches)
struct Flags {
  unsigned int bar[2];  // grid barrier (counter returns to 0, generation grows)
  unsigned int ticket;
  unsigned int pad[29];
  unsigned int fdone[MAXNB];
  unsigned int cnt[MAXNB * MAXNB];
  unsigned int pdone[MAXNB * MAXNB];
  unsigned int vdone[MAXNB * MAXNB];
};
constexpr size_t FLAGS_BYTES = (sizeof(Flags) + 4095) / 4096 * 4096;

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// thread 0 waits until *f >= want
__device__ __forceinline__ void wait_ge(const unsigned int* f, unsigned int want) {
  if (ld_acquire(f) >= want) return;
  while (ld_acquire(f) < want) __nanosleep(20);
}

// all threads' stores of this task, then the flag (release at GPU scope)
__device__ __forceinline__ void publish(unsigned int* f, unsigned int v) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
  }
}

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

// ---- block movement: global <-> shared (row-major, pitch PD) ----

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// issue the copies of one 64x64 block (8 x 16 B per thread); the caller commits/waits
__device__ __forceinline__ void load_async(double (*dst)[PD], const double* src, long long ld) {
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * THREADS;  // 16-byte chunk: row e >> 5, columns 2 (e & 31) ..
    cp_async16(&dst[e >> 5][2 * (e & 31)], src + (e >> 5) * ld + 2 * (e & 31));
  }
}

__device__ __forceinline__ void load_block(double (*dst)[PD], const double* src, long long ld) {
  load_async(dst, src, ld);
  cp_commit();
  cp_wait_all();
  __syncthreads();
}

// shared block -> global (coalesced 16-byte stores); lower_only: c <= r
__device__ __forceinline__ void store_block(double* dst, long long ld, const double (*src)[PD], bool lower_only) {
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = threadIdx.x + u * THREADS;
    const int r = e >> 5, c = 2 * (e & 31);
    const double2 v = *reinterpret_cast<const double2*>(&src[r][c]);
    if (!lower_only || c + 1 <= r) {
      *reinterpret_cast<double2*>(dst + r * ld + c) = v;
    } else if (c <= r) {
      dst[r * ld + c] = v.x;
    }
  }
}

// ---- 64x64x64 products on DMMA ----
// Warp w: rows 32 (w >> 2) .., columns 16 (w & 3) ..: 4 x 2 fragments of 8 x 8.
// Thread (g = lane >> 2, t = lane & 3) holds C[m0 + 8fm + g][n0 + 8fn + 2t (+1)].
struct Frag {
  double v[4][2][2];
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void frag_zero(Frag& f) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) f.v[i][j][0] = f.v[i][j][1] = 0.0;
}

// f += A B^T, A and B row-major [64][64] in shared memory (C[m][n] = sum_k A[m][k] B[n][k])
__device__ __forceinline__ void mm_nt(Frag& f, const double (*A)[PD], const double (*B)[PD]) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = 32 * (w >> 2), n0 = 16 * (w & 3);
#pragma unroll 4
  for (int k = 0; k < T; k += 4) {
    double a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = A[m0 + 8 * i + g][k + t];
#pragma unroll
    for (int j = 0; j < 2; ++j) b[j] = B[n0 + 8 * j + g][k + t];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma(f.v[i][j][0], f.v[i][j][1], a[i], b[j]);
  }
}

// f += A B, A and B row-major [64][64] (C[m][n] = sum_k A[m][k] B[k][n]); the B
// fragment reads are 2-way bank conflicted (only V's first term uses this)
__device__ __forceinline__ void mm_nn(Frag& f, const double (*A)[PD], const double (*B)[PD]) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = 32 * (w >> 2), n0 = 16 * (w & 3);
#pragma unroll 4
  for (int k = 0; k < T; k += 4) {
    double a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = A[m0 + 8 * i + g][k + t];
#pragma unroll
    for (int j = 0; j < 2; ++j) b[j] = B[k + t][n0 + 8 * j + g];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma(f.v[i][j][0], f.v[i][j][1], a[i], b[j]);
  }
}

// dst[m][n] = s * f (trans: dst[n][m])
__device__ __forceinline__ void frag_store(double (*dst)[PD], const Frag& f, double s, bool trans) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = 32 * (w >> 2), n0 = 16 * (w & 3);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int m = m0 + 8 * i + g, n = n0 + 8 * j + 2 * t;
      if (trans) {
        dst[n][m] = s * f.v[i][j][0];
        dst[n + 1][m] = s * f.v[i][j][1];
      } else {
        *reinterpret_cast<double2*>(&dst[m][n]) = make_double2(s * f.v[i][j][0], s * f.v[i][j][1]);
      }
    }
}

// dst[m][n] -= f (in place: every element belongs to one thread)
__device__ __forceinline__ void frag_sub_from(double (*dst)[PD], const Frag& f) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = 32 * (w >> 2), n0 = 16 * (w & 3);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      double2* p = reinterpret_cast<double2*>(&dst[m0 + 8 * i + g][n0 + 8 * j + 2 * t]);
      const double2 o = *p;
      *p = make_double2(o.x - f.v[i][j][0], o.y - f.v[i][j][1]);
    }
}

// ---- the 64x64 factor-and-invert on 4x4 register patches ----

// The chain's 4x4 patches: threads 0..135 own the lower patches (P, Q), Q <= P
// of the 16 x 16 patch grid (row-major enumeration); threads 136..255 own the 120
// strictly upper patches, which F never touches (they only write zeros where a
// full block is stored).  Halves F's per-pivot instruction stream against a
// 16 x 16 thread grid whose upper half computes garbage.
struct Patch {
  int P, Q;
  bool lower;
};

__device__ __forceinline__ Patch my_patch() {
  const int e = threadIdx.x;
  Patch pt;
  if (e < 136) {
    int r = static_cast<int>((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
    while ((r + 1) * (r + 2) / 2 <= e) ++r;
    while (r * (r + 1) / 2 > e) --r;
    pt.P = r;
    pt.Q = e - r * (r + 1) / 2;
    pt.lower = true;
  } else {
    // upper patch u = e - 136 of 120: row P has 15 - P of them (columns P+1..15)
    int u = e - 136, P = 0;
    while (u >= 15 - P) {
      u -= 15 - P;
      ++P;
    }
    pt.P = P;
    pt.Q = P + 1 + u;
    pt.lower = false;
  }
  return pt;
}

__device__ __forceinline__ void patch_load(double a[4][4], const double (*src)[PD], const Patch& pt) {
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const double2 v0 = *reinterpret_cast<const double2*>(&src[4 * pt.P + r][4 * pt.Q]);
    const double2 v1 = *reinterpret_cast<const double2*>(&src[4 * pt.P + r][4 * pt.Q + 2]);
    a[r][0] = v0.x;
    a[r][1] = v0.y;
    a[r][2] = v1.x;
    a[r][3] = v1.y;
  }
}

// lower patches store a; upper patches store zeros (zero_upper) or nothing
__device__ __forceinline__ void patch_store(double (*dst)[PD], const double a[4][4], const Patch& pt,
                                            bool zero_upper) {
  if (!pt.lower && !zero_upper) return;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const double2 v0 = pt.lower ? make_double2(a[r][0], a[r][1]) : make_double2(0.0, 0.0);
    const double2 v1 = pt.lower ? make_double2(a[r][2], a[r][3]) : make_double2(0.0, 0.0);
    *reinterpret_cast<double2*>(&dst[4 * pt.P + r][4 * pt.Q]) = v0;
    *reinterpret_cast<double2*>(&dst[4 * pt.P + r][4 * pt.Q + 2]) = v1;
  }
}

// 1/sqrt(d) and 1/d to ~1 ulp: MUFU seeds (~2^-22), then ONE cubic correction
// each -- y (1 + e/2 + 3e^2/8), e = 1 - d y^2, and y (1 + e + e^2), e = 1 - d y:
// four and three dependent FP64 ops (FP64 latency is ~23 cycles on B200,
// tools/micro/lat.cu), the two chains side by side
__device__ __forceinline__ double rsqrt_refined(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double u = d * y;
  const double e = fma(-u, y, 1.0);
  const double q = fma(e, 0.375, 0.5);
  const double w = y * e;
  return fma(w, q, y);
}

__device__ __forceinline__ double rcp_refined(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double e = fma(-d, y, 1.0);
  const double t = fma(e, e, e);
  return fma(y, t, y);
}

__device__ __forceinline__ void sts_f64(double* p, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))), "d"(v)
               : "memory");
}

// a (Schur complement, lower patches) -> L; x <- inv(L).  s.bad: 1-based first
// non-positive pivot (0 if none).  Pivot j (d = a_jj), for the owner of patch (P, Q):
//   a_rc -= a_rj a_cj / d      for c > j     (predicated, no selects)
//   X~_rc -= a_rj X~_jc / d    for r > j
// and column j of a / row j of X~ simply stop changing: the square roots are
// deferred -- L_ij = a_ij rs_j, X_jc = X~_jc rs_j with rs_j = 1/sqrt(d_j), applied
// once after the last pivot -- so the per-pivot critical path is only: barrier
// -> shared loads -> 1/d (MUFU + 3 FP64) -> the next column's update -> its
// publication.  The row buffers start zeroed, and X~ rows are zero right of
// their diagonal, so unpublished columns read as the zeros they are.
__device__ __forceinline__ void factor_inv64(Smem& s, double a[4][4], double x[4][4], const Patch& pt) {
  const int tid = threadIdx.x;
  const int P = pt.P, Q = pt.Q;
  int wrow = pt.lower ? 4 * P + 3 : -1;  // last row of this warp's lower patches
  wrow = __reduce_max_sync(0xffffffffu, wrow);
  int bad = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) x[r][c] = (4 * P + r == 4 * Q + c) ? 1.0 : 0.0;
  if (tid < 2 * T) (&s.row[0][0])[tid] = 0.0;
  __syncthreads();
  if (pt.lower && Q == 0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) s.col[0][4 * P + r] = a[r][0];
  }
  if (pt.lower && P == 0) {
#pragma unroll
    for (int c = 0; c < 4; ++c) s.row[0][4 * Q + c] = x[0][c];
  }
#pragma unroll 1
  for (int jb = 0; jb < T / 4; ++jb) {
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = 4 * jb + jj;
      const int buf = jj & 1;  // j & 1
      __syncthreads();
      if (tid >= 224) {  // warp 7 holds upper patches only: it does the square roots
        if (tid == 224) {
          const double dj = s.col[buf][j];
          s.rsv[j] = rsqrt_refined(dj);
          if (!(dj > 0.0) && bad == 0) bad = j + 1;
        }
        continue;
      }
      if (wrow < j) continue;  // every row of this warp is finished
      const double d = s.col[buf][j];
      const double2 cr01 = *reinterpret_cast<const double2*>(&s.col[buf][4 * P]);
      const double2 cr23 = *reinterpret_cast<const double2*>(&s.col[buf][4 * P + 2]);
      const double2 cc01 = *reinterpret_cast<const double2*>(&s.col[buf][4 * Q]);
      const double2 cc23 = *reinterpret_cast<const double2*>(&s.col[buf][4 * Q + 2]);
      const double2 rw01 = *reinterpret_cast<const double2*>(&s.row[buf][4 * Q]);
      const double2 rw23 = *reinterpret_cast<const double2*>(&s.row[buf][4 * Q + 2]);
      const double r2 = rcp_refined(d);
      if (!pt.lower) continue;
      const double crv[4] = {cr01.x, cr01.y, cr23.x, cr23.y};
      const double ccv[4] = {cc01.x, cc01.y, cc23.x, cc23.y};
      const double rwv[4] = {rw01.x, rw01.y, rw23.x, rw23.y};
      const int nj = (jj + 1) & 3;
      const int nb4 = jb + (jj == 3 ? 1 : 0);
      // the next pivot's column and X~ row first (one FMA after 1/d), published
      // before the rest
      if (4 * Q + nj > j) {
#pragma unroll
        for (int r = 0; r < 4; ++r) a[r][nj] = fma(-(crv[r] * ccv[nj]), r2, a[r][nj]);
      }
      if (4 * P + nj > j) {
#pragma unroll
        for (int c = 0; c < 4; ++c) x[nj][c] = fma(-(crv[nj] * rwv[c]), r2, x[nj][c]);
      }
      if (j + 1 < T) {
        if (Q == nb4) {
#pragma unroll
          for (int r = 0; r < 4; ++r) sts_f64(&s.col[buf ^ 1][4 * P + r], a[r][nj]);
        }
        if (P == nb4) {
#pragma unroll
          for (int c = 0; c < 4; ++c) sts_f64(&s.row[buf ^ 1][4 * Q + c], x[nj][c]);
        }
      }
      double lr[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) lr[r] = crv[r] * r2;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c == nj) continue;
        if (4 * Q + c > j) {
#pragma unroll
          for (int r = 0; r < 4; ++r) a[r][c] = fma(-lr[r], ccv[c], a[r][c]);
        }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (r == nj) continue;
        if (4 * P + r > j) {
#pragma unroll
          for (int c = 0; c < 4; ++c) x[r][c] = fma(-lr[r], rwv[c], x[r][c]);
        }
      }
    }
  }
  if (tid == 224) s.bad = bad;
  __syncthreads();
  // the deferred square roots: column scales for L, row scales for X
  if (pt.lower) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double sc = s.rsv[4 * Q + c];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r][c] *= sc;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const double sr = s.rsv[4 * P + r];
#pragma unroll
      for (int c = 0; c < 4; ++c) x[r][c] *= sr;
    }
  }
}

struct FlowArgs {
  double* A;
  long long lda;
  int nb;
  int mode;  // store_inv 0 / 1 / 2
  int* info;
  Flags* fl;
  double* xs;  // nb blocks of 64x64: X_kk = inv(L_kk), row-major
};

__device__ __forceinline__ double* blk(const FlowArgs& g, int i, int j) {
  return g.A + static_cast<long long>(i) * T * g.lda + static_cast<long long>(j) * T;
}
__device__ __forceinline__ double* xblk(const FlowArgs& g, int k) { return g.xs + static_cast<long long>(k) * T * T; }

// queue sizes of step k (k = 0 .. nb-2)
__device__ __forceinline__ int q_p(int nb, int k) { return nb - 2 - k; }
__device__ __forceinline__ int q_u(int nb, int k) { return (nb - 1 - k) * (nb - k) / 2 - 1; }
__device__ __forceinline__ int q_v(int mode, int k) { return mode == 2 ? k + 1 : 0; }

__device__ __forceinline__ int tri_root(int w) {
  int r = static_cast<int>((sqrtf(8.0f * w + 1.0f) - 1.0f) * 0.5f);
  while ((r + 1) * (r + 2) / 2 <= w) ++r;
  while (r * (r + 1) / 2 > w) --r;
  return r;
}

__device__ void do_P(const FlowArgs& g, Smem& s, int i, int k) {
  Flags* fl = g.fl;
  if (threadIdx.x == 0) {
    wait_ge(&fl->fdone[k], 1);
    wait_ge(&fl->cnt[i * MAXNB + k], k);
  }
  __syncthreads();
  load_async(s.a, blk(g, i, k), g.lda);
  load_async(s.b, xblk(g, k), T);  // B[n][q] = X[n][q]: C = A X^T
  cp_commit();
  cp_wait_all();
  __syncthreads();
  Frag f;
  frag_zero(f);
  mm_nt(f, s.a, s.b);
  frag_store(s.c, f, 1.0, false);
  __syncthreads();
  store_block(blk(g, i, k), g.lda, s.c, false);
  publish(&fl->pdone[i * MAXNB + k], 1);
  __syncthreads();
}

__device__ void do_U(const FlowArgs& g, Smem& s, int i, int j, int k) {
  Flags* fl = g.fl;
  if (threadIdx.x == 0) {
    wait_ge(&fl->pdone[i * MAXNB + k], 1);
    wait_ge(&fl->pdone[j * MAXNB + k], 1);
    wait_ge(&fl->cnt[i * MAXNB + j], k);
  }
  __syncthreads();
  load_async(s.a, blk(g, i, k), g.lda);
  if (j != i) load_async(s.b, blk(g, j, k), g.lda);
  load_async(s.c, blk(g, i, j), g.lda);
  cp_commit();
  cp_wait_all();
  __syncthreads();
  Frag f;
  frag_zero(f);
  mm_nt(f, s.a, j != i ? s.b : s.a);
  frag_sub_from(s.c, f);
  __syncthreads();
  store_block(blk(g, i, j), g.lda, s.c, i == j);
  publish(&fl->cnt[i * MAXNB + j], k + 1);
  __syncthreads();
}

// X_ik (i > k) of the full inverse, stored transposed into A's upper block (k, i)
__device__ void do_V(const FlowArgs& g, Smem& s, int i, int k) {
  Flags* fl = g.fl;
  Frag f;
  frag_zero(f);
  auto term = [&](int m) {  // f += L_im X_mk
    load_async(s.a, blk(g, i, m), g.lda);
    // m == k: X_kk row-major from the workspace (NN); else X_mk^T, which the upper
    // block (k, m) holds (NT)
    load_async(s.b, m == k ? xblk(g, k) : blk(g, k, m), m == k ? T : g.lda);
    cp_commit();
    cp_wait_all();
    __syncthreads();
    if (m == k)
      mm_nn(f, s.a, s.b);
    else
      mm_nt(f, s.a, s.b);
    __syncthreads();
  };
  if (i - 2 >= k) {  // the terms available before F(i): m = k .. i-2
    if (threadIdx.x == 0) {
      wait_ge(&fl->pdone[i * MAXNB + (i - 2)], 1);
      if (i - 2 > k) wait_ge(&fl->vdone[(i - 2) * MAXNB + k], 1);
      else wait_ge(&fl->fdone[k], 1);
    }
    __syncthreads();
    for (int m = k; m <= i - 2; ++m) term(m);
  }
  if (threadIdx.x == 0) {
    wait_ge(&fl->fdone[i], 1);
    if (i - 1 > k) wait_ge(&fl->vdone[(i - 1) * MAXNB + k], 1);
  }
  __syncthreads();
  term(i - 1);
  // X_ik = -X_ii S:  A operand X_ii (row-major), B operand S^T
  frag_store(s.b, f, 1.0, true);
  load_block(s.a, xblk(g, i), T);  // includes the barrier
  Frag y;
  frag_zero(y);
  mm_nt(y, s.a, s.b);
  frag_store(s.c, y, -1.0, true);  // c[n][m] = X_ik[m][n]: the transposed block
  __syncthreads();
  store_block(blk(g, k, i), g.lda, s.c, false);
  publish(&fl->vdone[i * MAXNB + k], 1);
  __syncthreads();
}

__global__ void __launch_bounds__(THREADS, 1) potrf_flow_kernel(const __grid_constant__ FlowArgs g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x;
  const int nb = g.nb;
  Flags* fl = g.fl;
  if (tid == 0) {
    int o = 0;
    for (int k = 0; k + 1 < nb; ++k) {
      s.off[k] = o;
      o += q_p(nb, k) + q_u(nb, k) + q_v(g.mode, k);
    }
    s.off[nb > 1 ? nb - 1 : 0] = o;
  }
  __syncthreads();
  const int total = s.off[nb > 1 ? nb - 1 : 0];

  if (blockIdx.x == 0) {
    // ---- the panel chain ----
    double a[4][4], x[4][4];
    const Patch pt = my_patch();
    load_block(s.c, blk(g, 0, 0), g.lda);
    if (pt.lower) patch_load(a, s.c, pt);
    for (int k = 0;; ++k) {
      // prefetch A_{k+1,k} (-> s.a) and A_{k+1,k+1} (-> s.d) under F when their
      // earlier updates are already in (the usual case)
      if (tid == 0)
        s.pre = (k + 1 < nb && ld_acquire(&fl->cnt[(k + 1) * MAXNB + k]) >= static_cast<unsigned>(k) &&
                 ld_acquire(&fl->cnt[(k + 1) * MAXNB + k + 1]) >= static_cast<unsigned>(k))
                    ? 1
                    : 0;
      __syncthreads();
      const bool pre = s.pre != 0;
      if (pre) {
        load_async(s.a, blk(g, k + 1, k), g.lda);
        load_async(s.d, blk(g, k + 1, k + 1), g.lda);
        cp_commit();
      }
      prof(k, 0);
      factor_inv64(s, a, x, pt);
      prof(k, 1);
      if (tid == 0 && s.bad && g.info && *reinterpret_cast<volatile int*>(g.info) == 0)
        *reinterpret_cast<volatile int*>(g.info) = k * T + s.bad;
      // X_kk -> s.b (row-major: the B operand of P), L_kk -> s.c; their global
      // stores (workspace X_kk, the tile's L_kk and inv(L_kk)^T) are issued now and
      // drain under P's product; ONE fence then publishes fdone[k] together with
      // pdone[k+1][k] (the queue's P(i,k) tasks have slack: their first consumer
      // on the chain is P(k+2,k+1), a step later)
      patch_store(s.b, x, pt, true);
      patch_store(s.c, a, pt, false);
      __syncthreads();
      store_block(xblk(g, k), T, s.b, false);
      store_block(blk(g, k, k), g.lda, s.c, true);
      if (g.mode >= 1) {
        double* Akk = blk(g, k, k);
        for (int e = tid; e < T * T; e += THREADS) {
          const int p = e >> 6, q = e & 63;
          if (p < q) Akk[p * g.lda + q] = s.b[q][p];
        }
      }
      prof(k, 2);
      if (k + 1 == nb) {
        publish(&fl->fdone[k], 1);
        break;
      }
      // ---- P(k+1, k) ----
      if (!pre) {
        if (tid == 0) wait_ge(&fl->cnt[(k + 1) * MAXNB + k], k);
        __syncthreads();
        load_async(s.a, blk(g, k + 1, k), g.lda);
        cp_commit();
      }
      cp_wait_all();
      __syncthreads();
      prof(k, 3);
      Frag f;
      frag_zero(f);
      mm_nt(f, s.a, s.b);
      __syncthreads();                 // s.c (L_kk staging) is free again
      frag_store(s.c, f, 1.0, false);  // L_{k+1,k}, row-major
      __syncthreads();
      store_block(blk(g, k + 1, k), g.lda, s.c, false);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&fl->fdone[k]), "r"(1u) : "memory");
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&fl->pdone[(k + 1) * MAXNB + k]), "r"(1u)
                     : "memory");
      }
      prof(k, 4);
      // ---- U(k+1, k+1, k): a = A_{k+1,k+1} - L L^T, never written back ----
      if (!pre) {
        if (tid == 0) wait_ge(&fl->cnt[(k + 1) * MAXNB + (k + 1)], k);
        __syncthreads();
        load_async(s.d, blk(g, k + 1, k + 1), g.lda);
        cp_commit();
      }
      prof(k, 5);
      frag_zero(f);
      mm_nt(f, s.c, s.c);
      cp_wait_all();
      __syncthreads();
      prof(k, 6);
      frag_sub_from(s.d, f);
      __syncthreads();
      if (pt.lower) patch_load(a, s.d, pt);
      __syncthreads();
      prof(k, 7);
    }
  }
  // ---- the queue (CTA 0 joins once the chain is done) ----
  while (true) {
    if (tid == 0) s.item = static_cast<int>(atomicAdd(&fl->ticket, 1u));
    __syncthreads();
    const int t = s.item;
    __syncthreads();
    if (t >= total) break;
    int k = 0;
    while (s.off[k + 1] <= t) ++k;
    const int idx = t - s.off[k];
    const int np = q_p(nb, k), nu = q_u(nb, k);
    if (idx < np) {
      do_P(g, s, k + 2 + idx, k);
    } else if (idx < np + nu) {
      const int w = idx - np + 1;  // local lower triangle of rows/cols k+1.., row-major, (0,0) skipped
      const int ii = tri_root(w), jj = w - ii * (ii + 1) / 2;
      do_U(g, s, k + 1 + ii, k + 1 + jj, k);
    } else {
      do_V(g, s, k + 1, idx - np - nu);
    }
  }
  // ---- every task is done: clear the flags for the next launch ----
  grid_barrier(fl->bar);
  const int words = static_cast<int>((sizeof(Flags) - offsetof(Flags, ticket)) / 4);
  unsigned int* w0 = &fl->ticket;
  for (int e = blockIdx.x * THREADS + tid; e < words; e += gridDim.x * THREADS) w0[e] = 0u;
}

}  // namespace

bool flow_supported(int n) { return n % T == 0 && n >= T && n / T <= MAXNB; }

size_t flow_workspace_bytes(int n) {
  return FLAGS_BYTES + static_cast<size_t>(n / T) * T * T * sizeof(double);
}

cudaError_t launch_dpotrf_flow(double* A, long long lda, int n, int* info, void* workspace, size_t ws_bytes,
                               cudaStream_t s, int store_inv) {
  if (!flow_supported(n) || ws_bytes < flow_workspace_bytes(n) || (lda % 2) ||
      (reinterpret_cast<uintptr_t>(A) & 15))
    return cudaErrorInvalidValue;
  static bool attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(potrf_flow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr[dev & 63] = true;
  }
  FlowArgs g;
  g.A = A;
  g.lda = lda;
  g.nb = n / T;
  g.mode = store_inv;
  g.info = info;
  // flags at the TOP of the (zero-initialised) stream scratch, whose bottom the
  // other cooperative kernels use; the X_kk blocks right below them
  char* top = static_cast<char*>(workspace) + (ws_bytes & ~size_t(4095));
  g.fl = reinterpret_cast<Flags*>(top - FLAGS_BYTES);
  g.xs = reinterpret_cast<double*>(top - flow_workspace_bytes(n));
  // the chain CTA plus enough queue CTAs for the widest step (nb^2/2 blocks)
  int grid = g.nb * g.nb / 4 + 1;
  if (grid > 64) grid = 64;
  if (grid < 2) grid = 2;
  void* args[] = {&g};
  count_launch();
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(potrf_flow_kernel), dim3(grid), dim3(THREADS), args, SMEM,
                                     s);
}

}  // namespace sfx
