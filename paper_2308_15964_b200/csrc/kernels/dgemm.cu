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
//    3-stage TMA ring with full/empty mbarriers (+ a TMA-prefetched C tile),
//    1 producer warp + 8 DMMA warps
//    (warp tile 64 x 32 = 8 x 4 DMMA fragments).
//  * k-permutation: within a 16-wide K step, thread (g, t) of a DMMA uses the
//    true k = 4t + kk for mma sub-step kk.  A summation index may be permuted
//    freely as long as A and B agree, and this makes a thread's A (and B^T)
//    operands 4 consecutive doubles -> two conflict-free ld.shared.v2.f64 under
//    the 128B swizzle.
//  * FP64 has no tcgen05 kind, so there is no TMEM accumulator: accumulators
//    live in registers (64 doubles / thread).
#include <cstdio>
#include <cstdlib>
#include <cudaTypedefs.h>

#include <unordered_map>

#include "kernels.h"
#include "ptx.cuh"

namespace sfx {
namespace {

// NN B-operand layout.  Default (0): four LDS.64 per sub-step, 2-way bank
// conflicted.  1: column-permuted operands, two conflict-free LDS.128 per
// sub-step -- measured SLOWER on C2 (roofline frac 0.876-0.882 vs 0.903-0.908,
// tools/r2c_ab.sh; ncu: 1.3 M vs 5.1 M bank conflicts per launch but DMMA pipe
// 88.2 % vs 90.4 % of active cycles: the LDS path is not the limit, the k-pair
// swaps (FSEL) and the longer operand live ranges cost more).  Kept for A/B.
#ifndef SFX_NN_COLPERM
#define SFX_NN_COLPERM 0
#endif
constexpr bool NN_COLPERM = SFX_NN_COLPERM != 0;

#ifndef SFX_GEMM_STAGES
#define SFX_GEMM_STAGES 3
#endif
#ifndef SFX_GEMM_CBUF
#define SFX_GEMM_CBUF 1
#endif
constexpr int BM = 128, BN = 128, BK = 16, STAGES = SFX_GEMM_STAGES;
constexpr int CONSUMER_WARPS = 8;
// one producer warpgroup (4 warps, one elected TMA lane) + two DMMA warpgroups;
// setmaxnreg moves registers from the producer to the consumers (40 / 232).
constexpr int THREADS = (CONSUMER_WARPS + 4) * 32;
// TRI (full-inverse TRSM): the producer warpgroup's three spare warps mask each
// B stage that crosses the diagonal in shared memory (see the kernel)
constexpr int MASK_WARPS = 3;
constexpr int A_STAGE = BM * BK * 8;  // 16 KiB
constexpr int B_STAGE = BN * BK * 8;  // 16 KiB
// C prefetch buffer: the producer TMA-loads the next epilogue's C tile (8 boxes
// of 16 x 128 doubles, 128B swizzle) while the consumers are still in the
// mainloop, so the epilogue reads C from shared memory instead of waiting on HBM
constexpr int C_BUF = SFX_GEMM_CBUF ? BM * BN * 8 : 0;  // 128 KiB
constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) + C_BUF + 3 * STAGES * 8 + 24 + 1024;
static_assert(SMEM_BYTES <= 232448, "dynamic shared memory per CTA");

// One launch covers G independent tile tasks of identical shape (grouped
// launch): CTA blockIdx.x -> (task, output tile).  Each task carries its own
// TMA descriptors in the (large, __grid_constant__) parameter block.
struct alignas(64) GemmOperands {
  CUtensorMap a, b, c;  // c: only when GemmGroup::cpref
  double* C;
};

template <int G>
struct GemmGroup {
  GemmOperands t[G];
  long long ldc;
  int ntasks;
  int ksplit;  // > 1: split-K, partial products are atomically added into C (beta == 1)
  int tri_split;  // TRI only, > 0: K-weighted split into items of tri_split units (column tile bn's k-range
                  // is [0, (bn+1)*BN) under the triangular mask) is cut into bn+1
                  // slices of BN/BK k-steps, atomically added (beta == 1)
  int tri;     // NN only: B is an upper-triangular block with a reciprocal diagonal
               // (B[k][n] = 0 for k > n, 1/B[k][k] on the diagonal) -- the inverse
               // blocks a store_inverses DPOTRF leaves in its tile's upper triangle
  int M, N, K;
  int tiles_n, tiles_per_task;
  int lower;
  int cpref;  // C tiles of interior output tiles are prefetched by TMA (beta != 0, ksplit == 1, !lower)
  int zero;     // always 0 at run time (the compiler cannot know): see the stage release
  int stagger;  // warpgroup 1 starts this many k-steps behind warpgroup 0 (SFX_GEMM_STAGGER, 0: off)
  int release;  // stage release: 0 = data-dependent arrive (default), 1 = fence.acq_rel.cta (A/B experiments)
  int cstore;   // cpref epilogue: results written back into the C buffer and stored by TMA (per warp)
  double alpha, beta;
};

constexpr int GROUP_MAX = 32;

template <bool TRANS_B, int G, bool TRI>
__global__ void __launch_bounds__(THREADS, 1) dgemm_dmma_kernel(const __grid_constant__ GemmGroup<G> p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint8_t* sC = sB + STAGES * B_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sC + C_BUF);
  uint64_t* empty = full + STAGES;
  uint64_t* cfull = empty + STAGES;
  uint64_t* cempty = cfull + 1;
  uint64_t* stagger = cempty + 1;  // warpgroup 1 starts one k-step behind warpgroup 0
  uint64_t* mfull = stagger + 1;   // TRI: stage s masked by the producer warpgroup's spare warps

  // TRI split: per row of output tiles, column tile bn spans (bn+1) K-units of
  // BN/BK k-steps; it is cut into items of U = tri_split units (the last one
  // shorter when U does not divide bn+1): tri_full U-unit items per row, then
  // tri_part shorter ones
  const int U = p.tri_split > 0 ? p.tri_split : 1;
  int tri_full = 0, tri_part = 0;
  for (int c = 0; c < p.tiles_n; ++c) {
    tri_full += (c + 1) / U;
    tri_part += ((c + 1) % U) != 0;
  }
  const int tri_rows = p.ntasks * (p.tiles_per_task / p.tiles_n);
  const int total = p.tri_split ? tri_rows * (tri_full + tri_part) : p.ntasks * p.tiles_per_task * p.ksplit;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ktiles_all = (p.K + BK - 1) / BK;
  const int kchunk = (ktiles_all + p.ksplit - 1) / p.ksplit;

  // linear work index -> (task, m0, n0, k-slice); lower = triangular enumeration (bm >= bn)
  auto coords = [&](int lin, int& task, int& m0, int& n0, int& kt0, int& kt1) {
    if (TRI && p.tri_split) {
      // all full items of every row first (CTAs are dispatched in blockIdx order,
      // so the shorter items fill the tail)
      const int rows = p.tiles_per_task / p.tiles_n;
      int rb, bn, q;
      if (lin < tri_rows * tri_full) {
        rb = lin / tri_full;
        int f = lin - rb * tri_full;
        bn = 0;
        while (f >= (bn + 1) / U) {
          f -= (bn + 1) / U;
          ++bn;
        }
        q = f;  // units [qU, qU + U)
      } else {
        const int l2 = lin - tri_rows * tri_full;
        rb = l2 / tri_part;
        int f = l2 - rb * tri_part;
        bn = 0;
        while (((bn + 1) % U) == 0 || f-- > 0) ++bn;  // the f-th column with a remainder
        q = (bn + 1) / U;
      }
      task = rb / rows;
      const int bm = rb - task * rows;
      m0 = bm * BM;
      n0 = bn * BN;
      kt0 = q * U * (BN / BK);
      kt1 = min(min(ktiles_all, kt0 + U * (BN / BK)), (bn + 1) * (BN / BK));
      return;
    }
    const int ks = lin % p.ksplit;
    lin /= p.ksplit;
    kt0 = ks * kchunk;
    kt1 = min(ktiles_all, kt0 + kchunk);
    task = lin / p.tiles_per_task;
    const int tile = lin - task * p.tiles_per_task;
    int bm, bn;
    if (TRI && p.ksplit == 1) {
      // unsplit TRI product (grouped full-inverse TRSMs): column tile bn spans
      // (bn+1) K-units, so hand out the longest columns first over ALL tasks of
      // the launch (CTAs are dispatched in blockIdx order): the tail is short tiles
      const int rows = p.tiles_per_task / p.tiles_n;
      const int per_col = p.ntasks * rows;
      const int bnr = (task * p.tiles_per_task + tile) / per_col;
      const int rem = (task * p.tiles_per_task + tile) - bnr * per_col;
      bn = p.tiles_n - 1 - bnr;
      task = rem / rows;
      bm = rem - task * rows;
    } else if (p.lower) {
      bm = static_cast<int>((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
      while ((bm + 1) * (bm + 2) / 2 <= tile) ++bm;
      while (bm * (bm + 1) / 2 > tile) --bm;
      bn = tile - bm * (bm + 1) / 2;
    } else {
      bm = tile / p.tiles_n;
      bn = tile % p.tiles_n;
    }
    m0 = bm * BM;
    n0 = bn * BN;
    if (TRI) {  // upper-triangular B: k-tiles below the diagonal are zero, skip them
      kt1 = min(kt1, (n0 + BN + BK - 1) / BK);
      if (kt1 < kt0) kt1 = kt0;
    }
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], CONSUMER_WARPS);
    }
    ptx::mbar_init(cfull, 1);
    ptx::mbar_init(cempty, p.cstore ? CONSUMER_WARPS : CONSUMER_WARPS * 32);
    ptx::mbar_init(stagger, CONSUMER_WARPS / 2);
    if (TRI)
      for (int s = 0; s < STAGES; ++s) ptx::mbar_init(&mfull[s], MASK_WARPS);
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp >= CONSUMER_WARPS) {
    // ---- TMA producer warpgroup (one elected lane) ----
    // Persistent: the smem ring runs across this CTA's tiles, so the next
    // tile's operands stream in while the consumers finish the current one.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == CONSUMER_WARPS && lane == 0) {
      int it = 0, cn = 0;
      for (int lin = blockIdx.x; lin < total; lin += gridDim.x) {
        int task, m0, n0, kt0, kt1;
        coords(lin, task, m0, n0, kt0, kt1);
        const CUtensorMap* tmA = &p.t[task].a;
        const CUtensorMap* tmB = &p.t[task].b;
        ptx::prefetch_tmap(tmA);
        ptx::prefetch_tmap(tmB);
        // this tile's C goes into the prefetch buffer once the previous epilogue
        // released it: issued at k-step kt0 + STAGES (the consumers have begun this
        // tile, so the previous epilogue is over and cempty will not block), it has
        // the rest of the mainloop to land; issued after the last k-step (round 1)
        // it arrived late: the consumers' cfull waits were ~2 % of their time
        const bool want_c = p.cpref && m0 + BM <= p.M && n0 + BN <= p.N;
        const int kc = kt1 - kt0 > STAGES ? kt0 + STAGES : kt1;
        auto load_c = [&]() {
          if (cn > 0) ptx::mbar_wait(cempty, (cn - 1) & 1);
          ptx::mbar_arrive_expect_tx(cfull, C_BUF);
          const CUtensorMap* tmC = &p.t[task].c;
          // boxes of 16 columns x 64 rows (the TMA-store epilogue writes each warp's
          // 64 x 32 block back as two of them)
#pragma unroll
          for (int q = 0; q < BN / 16; ++q)
#pragma unroll
            for (int hh = 0; hh < BM / 64; ++hh)
              ptx::tma_load_2d(sC + q * (BM * 128) + hh * (64 * 128), tmC, n0 + 16 * q, m0 + 64 * hh, cfull);
          ++cn;
        };
        for (int kt = kt0; kt < kt1; ++kt, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) ptx::mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          if (want_c && kt == kc) load_c();
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
        if (want_c && kc == kt1) load_c();
      }
    } else if (TRI && warp > CONSUMER_WARPS) {
      // ---- TRI operand masking (full-inverse TRSM) ----
      // B is the POTRF tile carrying W = inv(L)^T in its strict upper triangle and
      // L below it.  The product needs W: on the k-steps that cross the diagonal,
      // entries with k > n become 0 and the diagonal L_nn becomes 1 / L_nn.  The
      // spare producer warps rewrite those entries of the landed stage in shared
      // memory (same 128B-swizzled box layout the consumers read) and release it
      // on mfull[s]; the consumers' operand path has no mask code (round 2: the
      // in-register mask cost the TRI kernel 544 B of spills and a reciprocal in
      // the DMMA loop).
      const int mt = (warp - CONSUMER_WARPS - 1) * 32 + lane;
      int it = 0;
      for (int lin = blockIdx.x; lin < total; lin += gridDim.x) {
        int task, m0, n0, kt0, kt1;
        coords(lin, task, m0, n0, kt0, kt1);
        for (int kt = kt0; kt < kt1; ++kt, ++it) {
          const int s = it % STAGES;
          ptx::mbar_wait(&full[s], (it / STAGES) & 1);
          const int j = kt * BK - n0;  // tile-relative k of the stage's first row
          if (j + BK > 0) {            // rows k = j + kk >= n exist for columns n < j + BK
            double* bst = reinterpret_cast<double*>(sB + s * B_STAGE);
            const int ncols = min(BN, j + BK);
            for (int e = mt; e < ncols * BK; e += MASK_WARPS * 32) {
              const int n = e >> 4, kk = e & (BK - 1);
              const int k = j + kk;
              if (k < n) continue;
              const int nn = n & 15;
              double* ptr = bst + (((n >> 4) * 2048 + kk * 128 + (((nn >> 1) ^ (kk & 7)) << 4)) >> 3) + (nn & 1);
              *ptr = k == n ? __drcp_rn(*ptr) : 0.0;
            }
            ptx::fence_proxy_async();  // generic writes before the stage's next TMA refill
          }
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&mfull[s]);
        }
      }
    }
    return;
  }

  // ---- DMMA consumers ----
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warp grid, warp tile 64 x 32
  const int g = lane >> 2, t = lane & 3;
  const int sw = (TRANS_B || !NN_COLPERM) ? 0 : (t >> 1);  // NN: k order within a pair (see the B loads)
  // output columns (within the warp's 32) of this thread's accumulator pair P =
  // 0..3 (two adjacent columns each): NT: fragment j = P, columns 8P + 2t (+1);
  // NN (column permutation of the B loads): columns 8t + 2P (+1), i.e. a row's 8
  // values of one thread are contiguous
#define PCOL(P) ((TRANS_B || !NN_COLPERM) ? 8 * (P) + 2 * t : 8 * t + 2 * (P))
#define ACCX(i, P) ((TRANS_B || !NN_COLPERM) ? acc[i][P][0] : acc[i][2 * ((P)&1)][(P) >> 1])
#define ACCY(i, P) ((TRANS_B || !NN_COLPERM) ? acc[i][P][1] : acc[i][2 * ((P)&1) + 1][(P) >> 1])
  int it = 0, cn = 0;
  // TMA-store epilogue: this warp's C-buffer release waits for its bulk store to
  // have read shared memory -- deferred to the next tile's first k-step, so the
  // warp goes straight back to its DMMAs
  bool cpend = false;
  auto release_c = [&]() {
    if (cpend) {
      if (lane == 0) {
        ptx::bulk_wait_read0();
        ptx::mbar_arrive(cempty);
      }
      cpend = false;
    }
  };
  for (int lin = blockIdx.x; lin < total; lin += gridDim.x) {
    int task, m0, n0, kt0, kt1;
    coords(lin, task, m0, n0, kt0, kt1);
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = kt0; kt < kt1; ++kt, ++it) {
      const int s = it % STAGES;
      // Staggered warpgroups: the two DMMA warpgroups (rows 0-63 / 64-127 of the
      // tile, one warp of each per SMSP) would otherwise reach every tile's
      // epilogue together and leave the DMMA pipe idle through it.  Warpgroup 1
      // starts once warpgroup 0 has finished its first k-step; the lag persists,
      // so each epilogue runs beside the other warpgroup's mainloop.
      if (it == p.stagger && wm == 0 && lane == 0 && p.stagger) ptx::mbar_arrive(stagger);
      if (it == 0 && wm == 1 && p.stagger) ptx::mbar_wait(stagger, 0);
      ptx::mbar_wait(TRI ? &mfull[s] : &full[s], (it / STAGES) & 1);  // TRI: landed AND masked
      release_c();
      if (TRI && kt * BK >= n0 + wn * 32 + 32) {
        // TRI: every B operand of this warp's columns is below the diagonal in
        // this k-step (exact zeros): no loads, no DMMAs, just release the stage
        if (lane == 0) ptx::mbar_arrive(&empty[s]);
        continue;
      }
      const uint32_t aS = ptx::smem_u32(sA) + s * A_STAGE;
      const uint32_t bS = ptx::smem_u32(sB) + s * B_STAGE;
      // operands (true k = sigma(t, h, e) = 4t + 2h + (e ^ sw)): ordered shared
      // loads; the DMMAs are not volatile, so ptxas can slide this half's DMMAs
      // past the next loads
      uint32_t dep = 0;  // OR of the high words of every operand loaded in the second half
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double a[8][2], b[4][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = wm * 64 + 8 * i + g;  // r % 8 == g
          const double2 v = ptx::lds128(aS + r * 128 + (((2 * t + h) ^ g) << 4));
          if (h == 1) dep |= static_cast<uint32_t>(__double2hiint(v.x));
          a[i][0] = sw ? v.y : v.x;
          a[i][1] = sw ? v.x : v.y;
        }
        if (TRANS_B) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = wn * 32 + 8 * j + g;
            const double2 v = ptx::lds128(bS + r * 128 + (((2 * t + h) ^ g) << 4));
            if (h == 1) dep |= static_cast<uint32_t>(__double2hiint(v.x));
            b[j][0] = v.x;
            b[j][1] = v.y;
          }
        } else if (!NN_COLPERM) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int n = wn * 32 + 8 * j + g;
            const int q = n >> 4, nn = n & 15;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int k = 4 * t + 2 * h + e;
              const double v = ptx::lds64(bS + q * 2048 + k * 128 + (((nn >> 1) ^ (k & 7)) << 4) + (nn & 1) * 8);
              if (h == 1) dep |= static_cast<uint32_t>(__double2hiint(v));
              b[j][e] = v;  // TRI: already masked in shared memory
            }
          }
        } else {
          // NN: B stored [K][N] in 16-column TMA boxes (128B swizzle).  Thread
          // (g, t) owns warp columns 4g..4g+3 (fragment j, local column c ->
          // warp column 4c + j), so its operands of one k are 4 consecutive
          // doubles: two LDS.128 per sub-step instead of four LDS.64.  Threads
          // t >= 2 take the two k of each pair in the opposite order (sw), which
          // puts the rows one quarter-warp reads on swizzle phases p ^ {0,1,4,5}:
          // no bank conflict.
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int k = 4 * t + 2 * h + (e ^ sw);
#pragma unroll
            for (int jp = 0; jp < 2; ++jp) {
              const int n = wn * 32 + 4 * g + 2 * jp;
              const int nn = n & 15;
              const double2 v = ptx::lds128(bS + (n >> 4) * 2048 + k * 128 + (((nn >> 1) ^ (k & 7)) << 4));
              if (h == 1) dep |= static_cast<uint32_t>(__double2hiint(v.x));
              b[2 * jp][e] = v.x;  // TRI: already masked in shared memory
              b[2 * jp + 1][e] = v.y;
            }
          }
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) ptx::dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i][e], b[j][e]);
          if (h == 1 && e == 0) {
            // Release the stage (one arrive per warp) only once every shared load
            // this warp issued from it has COMPLETED: an mbarrier arrive does not
            // wait for in-flight ld.shared results, and arriving right after the
            // last load let the producer's next TMA overwrite rows not yet read
            // (round 1: rows 56-63 of C tiles wrong by ~1e-4, only with 2 output
            // tiles per CTA; tools/c2_check.py).  The arrive's ADDRESS depends on
            // every operand loaded in this half (dep & zero == 0 at run time, but
            // the compiler cannot fold it), so the instruction computing it waits
            // on the warp's load scoreboards -- for all 32 lanes, scoreboards are
            // per warp -- and no fence is needed.  release == 1: the previous
            // fence.acq_rel.cta + __syncwarp variant (MEMBAR, also waits for the
            // epilogue's global stores), kept for A/B measurements.
            if (p.release == 1) {
              ptx::fence_cta();
              __syncwarp();
              if (lane == 0) ptx::mbar_arrive(&empty[s]);
            } else if (lane == 0) {
              ptx::mbar_arrive_addr(ptx::smem_u32(&empty[s]) + (dep & static_cast<uint32_t>(p.zero)));
            }
          }
        }
      }
    }

    // ---- epilogue: C = beta*C + alpha*acc ----
    // Interior tiles batch all 32 C loads before any FMA/store so the loads
    // overlap (one HBM round trip per tile instead of one per fragment).
    double* const Cbase = p.t[task].C;
    if (p.ksplit > 1 || (TRI && p.tri_split)) {
      // split-K partial sum: C += alpha * acc (beta == 1 enforced by the launcher)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = m0 + wm * 64 + 8 * i + g;
        if (row >= p.M) continue;
#pragma unroll
        for (int P = 0; P < 4; ++P) {
          const int col = n0 + wn * 32 + PCOL(P);
          double* cp = Cbase + static_cast<long long>(row) * p.ldc + col;
          if (col < p.N && (!p.lower || row >= col)) atomicAdd(cp, p.alpha * ACCX(i, P));
          if (col + 1 < p.N && (!p.lower || row >= col + 1)) atomicAdd(cp + 1, p.alpha * ACCY(i, P));
        }
      }
      continue;
    }
    const bool interior = !p.lower && m0 + BM <= p.M && n0 + BN <= p.N;
    if (interior && p.cpref) {
      // C from the prefetch buffer: element (r, c) of the tile sits in box q = c / 16
      // at r * 128 + (((c % 16) / 2) ^ (r % 8)) * 16 + (c % 2) * 8
      release_c();  // (a tile without k-steps)
      ptx::mbar_wait(cfull, cn & 1);
      const uint32_t cS = ptx::smem_u32(sC);
      if (p.cstore) {
        // results back into the buffer (each thread rewrites the elements it read),
        // then one lane stores the warp's two 16 x 64 boxes by TMA
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = wm * 64 + 8 * i + g;
#pragma unroll
          for (int P = 0; P < 4; ++P) {
            const int c = wn * 32 + PCOL(P);
            const uint32_t ad = cS + (c >> 4) * (BM * 128) + r * 128 + ((((c & 15) >> 1) ^ g) << 4);
            const double2 cv = ptx::lds128(ad);
            double2 v;
            v.x = fma(p.beta, cv.x, p.alpha * ACCX(i, P));
            v.y = fma(p.beta, cv.y, p.alpha * ACCY(i, P));
            ptx::sts128(ad, v);
          }
        }
        ptx::fence_proxy_async();  // generic-proxy writes -> visible to the TMA store
        __syncwarp();
        if (lane == 0) {
          const CUtensorMap* tmC = &p.t[task].c;
#pragma unroll
          for (int qq = 0; qq < 2; ++qq) {
            const int q = 2 * wn + qq;
            ptx::tma_store_2d(tmC, n0 + 16 * q, m0 + 64 * wm, cS + q * (BM * 128) + wm * (64 * 128));
          }
          ptx::bulk_commit();
        }
        cpend = true;
        ++cn;
        continue;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = wm * 64 + 8 * i + g;
#pragma unroll
        for (int P = 0; P < 4; ++P) {
          const int c = wn * 32 + PCOL(P);
          const double2 cv = ptx::lds128(cS + (c >> 4) * (BM * 128) + r * 128 + ((((c & 15) >> 1) ^ g) << 4));
          double2 v;
          v.x = fma(p.beta, cv.x, p.alpha * ACCX(i, P));
          v.y = fma(p.beta, cv.y, p.alpha * ACCY(i, P));
          *reinterpret_cast<double2*>(Cbase + static_cast<long long>(m0 + r) * p.ldc + n0 + c) = v;
        }
      }
      ptx::mbar_arrive(cempty);  // this thread's reads of the buffer are done
      ++cn;
      continue;
    }
    if (interior) {
#pragma unroll
      for (int half = 0; half < 4; ++half) {  // 4 x 8 fragments: loads in flight together, no spills
        double2 cv[2][4];
        if (p.beta != 0.0) {
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int P = 0; P < 4; ++P)
              cv[i][P] = *reinterpret_cast<const double2*>(
                  Cbase + static_cast<long long>(m0 + wm * 64 + 8 * (2 * half + i) + g) * p.ldc + n0 + wn * 32 +
                  PCOL(P));
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int P = 0; P < 4; ++P) {
            const int ii = 2 * half + i;
            double2 v;
            if (p.beta != 0.0) {
              v.x = fma(p.beta, cv[i][P].x, p.alpha * ACCX(ii, P));
              v.y = fma(p.beta, cv[i][P].y, p.alpha * ACCY(ii, P));
            } else {
              v.x = p.alpha * ACCX(ii, P);
              v.y = p.alpha * ACCY(ii, P);
            }
            *reinterpret_cast<double2*>(Cbase + static_cast<long long>(m0 + wm * 64 + 8 * ii + g) * p.ldc + n0 +
                                        wn * 32 + PCOL(P)) = v;
          }
      }
      continue;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = m0 + wm * 64 + 8 * i + g;
      if (row >= p.M) continue;
      double* crow = Cbase + static_cast<long long>(row) * p.ldc;
#pragma unroll
      for (int P = 0; P < 4; ++P) {
        const int col = n0 + wn * 32 + PCOL(P);
        const double x = ACCX(i, P), y = ACCY(i, P);
        const bool ok0 = col < p.N && (!p.lower || row >= col);
        const bool ok1 = col + 1 < p.N && (!p.lower || row >= col + 1);
        if (ok0 && ok1) {
          double2* cp = reinterpret_cast<double2*>(crow + col);
          double2 v;
          if (p.beta == 0.0) {
            v.x = p.alpha * x;
            v.y = p.alpha * y;
          } else {
            double2 o = *cp;
            v.x = fma(p.beta, o.x, p.alpha * x);
            v.y = fma(p.beta, o.y, p.alpha * y);
          }
          *cp = v;
        } else {
          if (ok0) crow[col] = (p.beta == 0.0 ? 0.0 : p.beta * crow[col]) + p.alpha * x;
          if (ok1) crow[col + 1] = (p.beta == 0.0 ? 0.0 : p.beta * crow[col + 1]) + p.alpha * y;
        }
      }
    }
  }
  // a CTA whose whole work is shorter than the stagger still releases warpgroup 1
  if (wm == 0 && lane == 0 && p.stagger && it <= p.stagger) ptx::mbar_arrive(stagger);
  // outstanding TMA stores read this CTA's shared memory: complete them before exit
  if (p.cstore && lane == 0) ptx::bulk_wait0();
#undef PCOL
#undef ACCX
#undef ACCY
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

}  // namespace

namespace {
thread_local bool t_deterministic = false;
}
void set_deterministic_launches(bool on) { t_deterministic = on; }
bool deterministic_launches() { return t_deterministic; }

// launch-configuration counters (sfx_gemm_paths): which kernel path ran, so the
// parity tests can prove that they exercised the benchmarked configuration
std::atomic<unsigned long long> g_gemm_paths[SFX_GEMM_PATHS];

namespace {

void count_gemm_path(bool cpref, int per, int ksplit, bool tri, bool lower, bool trans_b, int ntasks, int total) {
  auto add = [](int k, unsigned long long v) { g_gemm_paths[k].fetch_add(v, std::memory_order_relaxed); };
  add(SFX_GEMM_LAUNCHES, 1);
  add(SFX_GEMM_TASKS, static_cast<unsigned long long>(ntasks));
  add(SFX_GEMM_WORK_ITEMS, static_cast<unsigned long long>(total));
  if (cpref) add(SFX_GEMM_CPREF, 1);
  if (per >= 2) add(SFX_GEMM_MULTI_TILE, 1);
  if (cpref && per >= 2) add(SFX_GEMM_CPREF_MULTI_TILE, 1);
  if (ksplit > 1) add(SFX_GEMM_SPLITK, 1);
  if (tri) add(SFX_GEMM_TRI, 1);
  if (lower) add(SFX_GEMM_LOWER, 1);
  if (trans_b) add(SFX_GEMM_NT, 1); else add(SFX_GEMM_NN, 1);
}

int num_sms() {
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

// Output tiles per persistent CTA: 2 once the launch has at least two waves of
// tiles and short mainloops (K < 1024: the second tile's operands stream in under
// the first one's epilogue), else 1 so small launches still spread over every SM
// and long-K tiles (Cholesky updates, b = 1024) release their SMs at a finer
// grain for the concurrent launches of other streams (measured: C2 b=512 32.2 vs
// 31.7 TFLOP/s with 2 vs 1; C3 b=1024 28.8 vs 27.5 with 1 vs 2).
int tiles_per_cta(int total, int K) {
  static int forced = [] {
    const char* e = getenv("SFX_GEMM_TILES_PER_CTA");
    return e ? atoi(e) : 0;
  }();
  if (forced > 0) return forced;
  // up to 4 output tiles per persistent CTA once the launch has that many tiles
  // per SM: the operand ring and the staggered warpgroups carry from tile to tile
  // (a tile's epilogue under the next tile's mainloop).  Round 1 (no stagger):
  // 2 tiles for K < 1024, 1 above; round 2 (r3i/r3j): C2 2 -> 3-4 tiles 0.913 ->
  // 0.919-0.921, C3 1 -> 2-4 tiles 32.2 -> 32.5-32.6 TFLOP/s, C5 33.8 -> 34.2
  (void)K;
  const int sms = num_sms();
  return total >= 4 * sms ? 4 : total >= 3 * sms ? 3 : total >= 2 * sms ? 2 : 1;
}

template <bool TB, int G, bool TRI = false>
cudaError_t launch_group_t(const GemmDesc* d, int n, int M, int N, int K, double alpha, double beta, bool lower,
                           bool tri, cudaStream_t stream) {
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(dgemm_dmma_kernel<TB, G, TRI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
  // split-K decided below; the C prefetch needs beta != 0, no split and a full tile
  const bool want_cpref = C_BUF > 0 && beta != 0.0 && !lower && M >= BM && N >= BN;
  p.ldc = d[0].ldc;
  p.M = M;
  p.N = N;
  p.K = K;
  p.alpha = alpha;
  p.beta = beta;
  p.lower = lower ? 1 : 0;
  p.tri = tri ? 1 : 0;
  p.zero = 0;
  static const int release_mode = getenv("SFX_GEMM_RELEASE") ? atoi(getenv("SFX_GEMM_RELEASE")) : 0;
  p.release = release_mode;
  static const int stagger_mode = getenv("SFX_GEMM_STAGGER") ? atoi(getenv("SFX_GEMM_STAGGER")) : 1;
  // at most STAGES - 1: warpgroup 0 cannot run further ahead (every stage needs
  // both warpgroups' release before the producer refills it)
  p.stagger = stagger_mode < 0 ? 0 : (stagger_mode > STAGES - 1 ? STAGES - 1 : stagger_mode);
  const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  p.tiles_n = tn;
  p.tiles_per_task = lower ? tm * (tm + 1) / 2 : tm * tn;
  p.ntasks = n;
  // Small launches (the critical-path GEMMs inside TRSM/POTRF) split K so that
  // they still cover the SMs: each slice keeps >= 8 K-steps of 16.
  p.ksplit = 1;
  // the full-inverse TRSM (square TRI product, beta = 1 into a zeroed X): K-weighted
  // slices instead of a uniform split-K
  const bool det = deterministic_launches();
  p.tri_split = (!det && TRI && beta == 1.0 && N == K && N % BN == 0 && M % BM == 0) ? 1 : 0;
  if (beta == 1.0 && !p.tri_split && !det) {
    const int tiles = p.tiles_per_task * n, ksteps = (K + BK - 1) / BK;
    while (tiles * p.ksplit * 2 <= num_sms() && ksteps / (p.ksplit * 2) >= 8) p.ksplit *= 2;
  }
  // the C prefetch serves the direct epilogue only: split-K and TRI-split items
  // add into C with atomics and never read the buffer (with 2 tiles per CTA the
  // producer would then wait forever for the buffer's release)
  p.cpref = want_cpref && p.ksplit == 1 && !p.tri_split ? 1 : 0;
  if (p.cpref)
    for (int i = 0; i < n; ++i)
      if (!make_tmap_f64_2d(&p.t[i].c, d[i].C, N, M, d[i].ldc, 16, 64, true)) return cudaErrorInvalidValue;
  static const int cstore_mode = getenv("SFX_GEMM_TMA_STORE") ? atoi(getenv("SFX_GEMM_TMA_STORE")) : 0;
  p.cstore = p.cpref && cstore_mode ? 1 : 0;
  // K-weighted TRI split: one-unit items (BN/BK k-steps each), or two-unit items
  // (half the atomic epilogues) once one-unit items would fill the SMs more than
  // once over
  if (p.tri_split) {
    const int units = tm * n * (tn * (tn + 1) / 2);
    p.tri_split = units > num_sms() ? 2 : 1;
  }
  int tri_items = 0;  // per row of output tiles: full items + shorter items (see the kernel)
  for (int c = 0; c < tn; ++c) tri_items += (c + 1) / (p.tri_split ? p.tri_split : 1) +
                                          (((c + 1) % (p.tri_split ? p.tri_split : 1)) != 0);
  const int total = p.tri_split ? n * tm * tri_items : p.tiles_per_task * n * p.ksplit;
  // persistent CTAs, at most tiles_per_cta() output tiles each: the operand
  // ring streams the next tile during the epilogue, while SMs still free up
  // often enough for high-priority (critical-path) kernels to get in
  const int per = tiles_per_cta(total, K);
  const int grid = (total + per - 1) / per;
  count_launch();
  count_gemm_path(p.cpref != 0, per, p.tri_split ? 2 : p.ksplit, TRI, lower, TB, n, total);
  dgemm_dmma_kernel<TB, G, TRI><<<grid, THREADS, SMEM_BYTES, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_dgemm_group(const GemmDesc* d, int n, int M, int N, int K, double alpha, double beta,
                               bool trans_b, bool lower, cudaStream_t stream, bool tri) {
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
      e = trans_b ? launch_group_t<true, 1>(d + i0, 1, M, N, K, alpha, beta, lower, false, stream)
                  : (tri ? launch_group_t<false, 1, true>(d + i0, 1, M, N, K, alpha, beta, lower, true, stream)
                         : launch_group_t<false, 1>(d + i0, 1, M, N, K, alpha, beta, lower, false, stream));
    else
      e = trans_b ? launch_group_t<true, GROUP_MAX>(d + i0, m, M, N, K, alpha, beta, lower, false, stream)
                  : (tri ? launch_group_t<false, GROUP_MAX, true>(d + i0, m, M, N, K, alpha, beta, lower, true, stream)
                         : launch_group_t<false, GROUP_MAX>(d + i0, m, M, N, K, alpha, beta, lower, false, stream));
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
