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

struct GemmArgs {
  double* C;
  long long ldc;
  int M, N, K;
  int tiles_n;
  int lower;
  double alpha, beta;
};

template <bool TRANS_B>
__global__ void __launch_bounds__(THREADS, 1)
    dgemm_dmma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE);
  uint64_t* empty = full + STAGES;

  int bm, bn;
  if (p.lower) {
    // triangular enumeration of lower CTA tiles: idx -> (bm >= bn)
    int idx = blockIdx.x;
    bm = static_cast<int>((sqrtf(8.0f * idx + 1.0f) - 1.0f) * 0.5f);
    while ((bm + 1) * (bm + 2) / 2 <= idx) ++bm;
    while (bm * (bm + 1) / 2 > idx) --bm;
    bn = idx - bm * (bm + 1) / 2;
  } else {
    bm = blockIdx.x / p.tiles_n;
    bn = blockIdx.x % p.tiles_n;
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
      ptx::prefetch_tmap(&tmA);
      ptx::prefetch_tmap(&tmB);
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) ptx::mbar_wait(&empty[s], ((kt / STAGES) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&full[s], A_STAGE + B_STAGE);
        ptx::tma_load_2d(sA + s * A_STAGE, &tmA, kt * BK, m0, &full[s]);
        if (TRANS_B) {
          ptx::tma_load_2d(sB + s * B_STAGE, &tmB, kt * BK, n0, &full[s]);
        } else {
#pragma unroll
          for (int q = 0; q < BN / 16; ++q)
            ptx::tma_load_2d(sB + s * B_STAGE + q * 2048, &tmB, n0 + 16 * q, kt * BK, &full[s]);
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
    double* crow = p.C + static_cast<long long>(row) * p.ldc;
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

bool make_tmap_f64_2d(CUtensorMap* tm, const double* base, uint64_t inner, uint64_t outer, uint64_t ld,
                      uint32_t box_inner, uint32_t box_outer, bool swizzle128) {
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
  return r == CUDA_SUCCESS;
}

cudaError_t launch_dgemm(const double* A, long long lda, const double* B, long long ldb, double* C, long long ldc,
                         int M, int N, int K, double alpha, double beta, bool trans_b, bool lower,
                         cudaStream_t stream) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if ((lda & 1) || (ldb & 1) || (ldc & 1) || (reinterpret_cast<uintptr_t>(A) & 15) ||
      (reinterpret_cast<uintptr_t>(B) & 15) || (reinterpret_cast<uintptr_t>(C) & 15))
    return cudaErrorMisalignedAddress;
  if (K <= 0) {
    // C = beta*C: a degenerate update (no contraction), handled by the same epilogue
    // with alpha = 0 would still need operand loads; reject instead.
    return cudaErrorInvalidValue;
  }
  static bool attr_set[64][2] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63][trans_b]) {
    cudaError_t e = trans_b ? cudaFuncSetAttribute(dgemm_dmma_kernel<true>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES)
                            : cudaFuncSetAttribute(dgemm_dmma_kernel<false>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set[dev & 63][trans_b] = true;
  }
  CUtensorMap tmA, tmB;
  if (!make_tmap_f64_2d(&tmA, A, K, M, lda, BK, BM, true)) return cudaErrorInvalidValue;
  bool ok = trans_b ? make_tmap_f64_2d(&tmB, B, K, N, ldb, BK, BN, true)
                    : make_tmap_f64_2d(&tmB, B, N, K, ldb, 16, BK, true);
  if (!ok) return cudaErrorInvalidValue;
  GemmArgs p;
  p.C = C;
  p.ldc = ldc;
  p.M = M;
  p.N = N;
  p.K = K;
  p.alpha = alpha;
  p.beta = beta;
  p.lower = lower ? 1 : 0;
  const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  p.tiles_n = tn;
  const int grid = lower ? tm * (tm + 1) / 2 : tm * tn;
  if (trans_b)
    dgemm_dmma_kernel<true><<<grid, THREADS, SMEM_BYTES, stream>>>(tmA, tmB, p);
  else
    dgemm_dmma_kernel<false><<<grid, THREADS, SMEM_BYTES, stream>>>(tmA, tmB, p);
  return cudaGetLastError();
}

}  // namespace sfx
