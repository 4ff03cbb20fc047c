// Tile DGEMM / DSYRK on the FP64 tensor path (DMMA) with TMA-fed shared memory.
//
// C[M x N] = beta * C + alpha * A[M x K] * op(B)
//   op(B) = B^T with B stored [N x K] row-major   (trans_b = 1; Cholesky update
//           A_ij -= A_ik A_jk^T and DSYRK A_ii -= A_ik A_ik^T)
//   op(B) = B   with B stored [K x N] row-major   (trans_b = 0; tiled DGEMM
//           C_ij += A_ik B_kj)
// `lower` restricts both the CTA grid and the stores to row >= col (DSYRK).
//
// The reference has no tile bodies at all (SURVEY.md §2, row "Tile bodies ...
// absent"); the CPU restatement in oracle/bodies.py is the parity oracle.
//
// Design (B200, sm_100a):
//  * CTA tile 128 x 128, K-step 16 doubles (128 B rows -> 128B TMA swizzle),
//    4-stage TMA ring with full/empty mbarriers, 1 producer warp + 8 DMMA warps
//    (warp tile 64 x 32 = 8 x 4 DMMA fragments).
//  * k-permutation: within a 16-wide K step, thread (g, t) of a DMMA uses the
//    true k = 4t + kk for mma sub-step kk.  A summation index may be permuted
//    freely as long as A and B agree, and this makes a thread's A (and B^T)
//    operands 4 consecutive doubles -> two conflict-free ld.shared.v2.f64 under
//    the 128B swizzle.
//  * FP64 has no tcgen05 kind, so there is no TMEM accumulator: accumulators
//    live in registers (64 doubles / thread).
#include <cstdio>
#include <cudaTypedefs.h>

#include <unordered_map>

#include "kernels.h"
#include "ptx.cuh"

namespace sfx {
namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4;
constexpr int CONSUMER_WARPS = 8;
// one producer warpgroup (4 warps, one elected TMA lane) + two DMMA warpgroups;
// setmaxnreg moves registers from the producer to the consumers (40 / 232).
constexpr int THREADS = (CONSUMER_WARPS + 4) * 32;
constexpr int A_STAGE = BM * BK * 8;  // 16 KiB
constexpr int B_STAGE = BN * BK * 8;  // 16 KiB
constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) + 2 * STAGES * 8 + 1024;

// One launch covers G independent tile tasks of identical shape (grouped
// launch): CTA blockIdx.x -> (task, output tile).  Each task carries its own
// TMA descriptors in the (large, __grid_constant__) parameter block.
struct alignas(64) GemmOperands {
  CUtensorMap a, b;
  double* C;
};

template <int G>
struct GemmGroup {
  GemmOperands t[G];
  long long ldc;
  int M, N, K;
  int tiles_n, tiles_per_task;
  int lower;
  double alpha, beta;
};

constexpr int GROUP_MAX = 32;

template <bool TRANS_B, int G>
__global__ void __launch_bounds__(THREADS, 1) dgemm_dmma_kernel(const __grid_constant__ GemmGroup<G> p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE);
  uint64_t* empty = full + STAGES;

  const int task = blockIdx.x / p.tiles_per_task;
  const int tile = blockIdx.x - task * p.tiles_per_task;
  const CUtensorMap* tmA = &p.t[task].a;
  const CUtensorMap* tmB = &p.t[task].b;
  double* const Cbase = p.t[task].C;
  int bm, bn;
  if (p.lower) {
    // triangular enumeration of lower CTA tiles: idx -> (bm >= bn)
    int idx = tile;
    bm = static_cast<int>((sqrtf(8.0f * idx + 1.0f) - 1.0f) * 0.5f);
    while ((bm + 1) * (bm + 2) / 2 <= idx) ++bm;
    while (bm * (bm + 1) / 2 > idx) --bm;
    bn = idx - bm * (bm + 1) / 2;
  } else {
    bm = tile / p.tiles_n;
    bn = tile % p.tiles_n;
  }
  const int m0 = bm * BM, n0 = bn * BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ktiles = (p.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], CONSUMER_WARPS * 32);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp >= CONSUMER_WARPS) {
    // ---- TMA producer warpgroup (one elected lane) ----
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == CONSUMER_WARPS && lane == 0) {
      ptx::prefetch_tmap(tmA);
      ptx::prefetch_tmap(tmB);
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) ptx::mbar_wait(&empty[s], ((kt / STAGES) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&full[s], A_STAGE + B_STAGE);
        ptx::tma_load_2d(sA + s * A_STAGE, tmA, kt * BK, m0, &full[s]);
        if (TRANS_B) {
          ptx::tma_load_2d(sB + s * B_STAGE, tmB, kt * BK, n0, &full[s]);
        } else {
#pragma unroll
          for (int q = 0; q < BN / 16; ++q)
            ptx::tma_load_2d(sB + s * B_STAGE + q * 2048, tmB, n0 + 16 * q, kt * BK, &full[s]);
        }
      }
    }
    return;
  }

  // ---- DMMA consumers ----
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warp grid, warp tile 64 x 32
  const int g = lane >> 2, t = lane & 3;
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const uint32_t sA_u = ptx::smem_u32(sA), sB_u = ptx::smem_u32(sB);
  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % STAGES;
    ptx::mbar_wait(&full[s], (kt / STAGES) & 1);
    const uint32_t aBase = sA_u + s * A_STAGE;
    const uint32_t bBase = sB_u + s * B_STAGE;
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // k half: true k = 4t + 2h + {0,1}
      double a[8][2], b[4][2];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = wm * 64 + 8 * i + g;  // r % 8 == g
        double2 v = ptx::lds128(aBase + r * 128 + (((2 * t + h) ^ g) << 4));
        a[i][0] = v.x;
        a[i][1] = v.y;
      }
      if (TRANS_B) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = wn * 32 + 8 * j + g;
          double2 v = ptx::lds128(bBase + r * 128 + (((2 * t + h) ^ g) << 4));
          b[j][0] = v.x;
          b[j][1] = v.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int n = wn * 32 + 8 * j + g;
          const int q = n >> 4, nn = n & 15;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int k = 4 * t + 2 * h + e;
            b[j][e] = ptx::lds64(bBase + q * 2048 + k * 128 + ((((nn >> 1) ^ (k & 7))) << 4) + (nn & 1) * 8);
          }
        }
      }
      if (h == 1) ptx::mbar_arrive(&empty[s]);  // operands are in registers
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) ptx::dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i][e], b[j][e]);
    }
  }

  // ---- epilogue: C = beta*C + alpha*acc ----
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = m0 + wm * 64 + 8 * i + g;
    if (row >= p.M) continue;
    double* crow = Cbase + static_cast<long long>(row) * p.ldc;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = n0 + wn * 32 + 8 * j + 2 * t;
      const bool ok0 = col < p.N && (!p.lower || row >= col);
      const bool ok1 = col + 1 < p.N && (!p.lower || row >= col + 1);
      if (ok0 && ok1) {
        double2* cp = reinterpret_cast<double2*>(crow + col);
        double2 v;
        if (p.beta == 0.0) {
          v.x = p.alpha * acc[i][j][0];
          v.y = p.alpha * acc[i][j][1];
        } else {
          double2 o = *cp;
          v.x = fma(p.beta, o.x, p.alpha * acc[i][j][0]);
          v.y = fma(p.beta, o.y, p.alpha * acc[i][j][1]);
        }
        *cp = v;
      } else {
        if (ok0) crow[col] = (p.beta == 0.0 ? 0.0 : p.beta * crow[col]) + p.alpha * acc[i][j][0];
        if (ok1) crow[col + 1] = (p.beta == 0.0 ? 0.0 : p.beta * crow[col + 1]) + p.alpha * acc[i][j][1];
      }
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

}  // namespace

namespace {
struct TmapKey {
  const void* base;
  uint64_t inner, outer, ld;
  uint32_t bi, bo, sw;
  bool operator==(const TmapKey& o) const {
    return base == o.base && inner == o.inner && outer == o.outer && ld == o.ld && bi == o.bi && bo == o.bo &&
           sw == o.sw;
  }
};
struct TmapHash {
  size_t operator()(const TmapKey& k) const {
    size_t h = reinterpret_cast<size_t>(k.base) * 0x9E3779B97F4A7C15ull;
    h ^= (k.inner * 31 + k.outer) * 0xBF58476D1CE4E5B9ull + (k.ld << 7) + (k.bi << 3) + k.bo + k.sw;
    return h;
  }
};
}  // namespace

bool make_tmap_f64_2d(CUtensorMap* tm, const double* base, uint64_t inner, uint64_t outer, uint64_t ld,
                      uint32_t box_inner, uint32_t box_outer, bool swizzle128) {
  // Encoding a descriptor is a driver call of a few microseconds; tiles keep
  // their arena address while resident, so descriptors are cached per thread
  // (one executor thread per device).  The key holds every encode input, so a
  // hit is always exact even after the arena slot was reused.
  thread_local std::unordered_map<TmapKey, CUtensorMap, TmapHash> cache;
  const TmapKey key{base, inner, outer, ld, box_inner, box_outer, swizzle128 ? 1u : 0u};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *tm = it->second;
    return true;
  }
  auto enc = tmap_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * sizeof(double)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  if (cache.size() > (1u << 16)) cache.clear();
  cache.emplace(key, *tm);
  return true;
}

namespace {

template <bool TB, int G>
cudaError_t launch_group_t(const GemmDesc* d, int n, int M, int N, int K, double alpha, double beta, bool lower,
                           cudaStream_t stream) {
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(dgemm_dmma_kernel<TB, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set[dev & 63] = true;
  }
  GemmGroup<G> p;
  for (int i = 0; i < n; ++i) {
    if (!make_tmap_f64_2d(&p.t[i].a, d[i].A, K, M, d[i].lda, BK, BM, true)) return cudaErrorInvalidValue;
    const bool ok = TB ? make_tmap_f64_2d(&p.t[i].b, d[i].B, K, N, d[i].ldb, BK, BN, true)
                       : make_tmap_f64_2d(&p.t[i].b, d[i].B, N, K, d[i].ldb, 16, BK, true);
    if (!ok) return cudaErrorInvalidValue;
    p.t[i].C = d[i].C;
  }
  p.ldc = d[0].ldc;
  p.M = M;
  p.N = N;
  p.K = K;
  p.alpha = alpha;
  p.beta = beta;
  p.lower = lower ? 1 : 0;
  const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  p.tiles_n = tn;
  p.tiles_per_task = lower ? tm * (tm + 1) / 2 : tm * tn;
  count_launch();
  dgemm_dmma_kernel<TB, G><<<p.tiles_per_task * n, THREADS, SMEM_BYTES, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_dgemm_group(const GemmDesc* d, int n, int M, int N, int K, double alpha, double beta,
                               bool trans_b, bool lower, cudaStream_t stream) {
  if (M <= 0 || N <= 0 || n <= 0) return cudaSuccess;
  if (K <= 0) return cudaErrorInvalidValue;
  for (int i = 0; i < n; ++i) {
    if ((d[i].lda & 1) || (d[i].ldb & 1) || (d[i].ldc & 1) || (reinterpret_cast<uintptr_t>(d[i].A) & 15) ||
        (reinterpret_cast<uintptr_t>(d[i].B) & 15) || (reinterpret_cast<uintptr_t>(d[i].C) & 15) ||
        d[i].ldc != d[0].ldc)
      return cudaErrorMisalignedAddress;
  }
  for (int i0 = 0; i0 < n; i0 += GROUP_MAX) {
    const int m = n - i0 < GROUP_MAX ? n - i0 : GROUP_MAX;
    cudaError_t e;
    if (m == 1)
      e = trans_b ? launch_group_t<true, 1>(d + i0, 1, M, N, K, alpha, beta, lower, stream)
                  : launch_group_t<false, 1>(d + i0, 1, M, N, K, alpha, beta, lower, stream);
    else
      e = trans_b ? launch_group_t<true, GROUP_MAX>(d + i0, m, M, N, K, alpha, beta, lower, stream)
                  : launch_group_t<false, GROUP_MAX>(d + i0, m, M, N, K, alpha, beta, lower, stream);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_dgemm(const double* A, long long lda, const double* B, long long ldb, double* C, long long ldc,
                         int M, int N, int K, double alpha, double beta, bool trans_b, bool lower,
                         cudaStream_t stream) {
  GemmDesc d{A, lda, B, ldb, C, ldc};
  return launch_dgemm_group(&d, 1, M, N, K, alpha, beta, trans_b, lower, stream);
}

}  // namespace sfx
