// Particle-group P2P interaction kernel (FP64, sm_100a).
//
// Blocks are 4 x n SoA tiles: positions P = (x, y, z, q), accumulators
// F = (fx, fy, fz, pot).  For target a and source b (a != b):
//   r2   = |x_a - x_b|^2 + eps2
//   pot_a += q_b / r
//   F_a  += q_a q_b (x_a - x_b) / r^3
// (oracle/bodies.py _one_side / p2p_pair / p2p_self).  A pair task (i, j)
// owes every ORDERED interaction between the two groups (both directions),
// a self task every ordered pair a != b inside one group: N(N-1) in total,
// the unit of the metric.
//
// Mutual evaluation.  Both directions of a pair share dx, r2 and 1/r, so the
// kernel evaluates each UNORDERED pair once and applies it to both sides:
//   u = 1/r, pa = q_a u, pb = q_b u, s = pa pb u  (= q_a q_b / r^3)
//   pot_a += pb, pot_b += pa, F_a += s d, F_b -= s d       (d = x_a - x_b)
// = 3 DADD + 3 DFMA (r2) + MUFU.RSQ64H + 5 (one 3rd-order refinement step,
// full double) + 4 DMUL + 2 DADD + 6 DFMA = 23 FP64 ops per unordered pair,
// 11.5 per ordered interaction (the one-directional formulation needs 21).
//
// Layout (warp-shuffle rotation).  A CTA owns a BLK = 1024-target block of side
// a and a 1024-source block of side b; each of its 4 warps holds 256 targets in
// registers (TPT = 8 per lane, with their accumulators).  The b block is
// walked in chunks of 64: every lane loads SPT = 2 sources (coalesced) and
// zeroes their accumulators, then the warp does 32 rotation steps: evaluate
// the lane's 8 x 2 pairs, pass the 2 sources and their accumulators to the
// next lane (__shfl_sync: 32 32-bit shuffles per step, so TPT = 8 keeps the
// FP64 pipe -- 16 pairs x 23 instructions -- the bound, not the shuffle unit;
// with TPT = 4 the shuffles were).  After 32 steps every source has met all 256
// targets of the warp and is back on its home lane with its accumulated
// contributions; the 4 warps' partials are summed in shared memory and added
// to F_b with one FP64 atomic per component.  Targets flush their
// accumulators with FP64 atomics at the end.  Because every update of F is a
// device atomic, other CTAs of the same task and other tasks of the same
// commutative group may add into the same accumulators concurrently: the
// runtime takes these ops' commutative guards in shared mode
// (runtime.h accumulates_atomically) and groups up to 32 same-shape tasks
// into one launch (launch_p2p_group).
//
// Self task: the blocks (ba, bb) with bb >= ba of one group; on diagonal
// blocks only pairs with index(b) > index(a) count, so each unordered pair is
// evaluated once (the mask costs one compare + select, diagonal blocks only).
// Padding lanes (past n) carry q = 0 and a far-away position, contributing 0.
#include "kernels.h"

namespace sfx {
namespace {

constexpr int THREADS = 128;           // 4 warps
constexpr int TPT = 8;                 // targets per lane
constexpr int SPT = 2;                 // sources per lane per chunk
constexpr int BLK = 32 * TPT * (THREADS / 32);  // 1024: targets per CTA = sources per CTA
constexpr int CHUNK = 32 * SPT;        // 64 sources per rotation round
constexpr double FAR = 1e100;          // padding position (r2 ~ 1e200: finite, u ~ 1e-100)

// 1/sqrt(x), x > 0 normal: MUFU.RSQ64H seed refined by one third-order step
// y' = y + y e (1/2 + 3/8 e), e = 1 - x y^2 (error ~ (5/16) e^3: full double
// for a seed good to ~2^-22).  5 FP64 ops, no slow path.
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x * y, y, 1.0);
  const double c = fma(0.375, e, 0.5);
  return fma(y * e, c, y);
}

struct P2PArgs {
  const double* pa;  // 4 x na (ld_pa)
  const double* pb;  // 4 x nb (ld_pb)
  double* fa;
  double* fb;
  long long ld_pa, ld_pb, ld_fa, ld_fb;
  int na, nb;
  int nblk_a, nblk_b;  // blocks of BLK along a and b
  double eps2;
};

template <bool DIAG>
__device__ __forceinline__ void pair_step(const double (&xa)[TPT], const double (&ya)[TPT], const double (&za)[TPT],
                                          const double (&qa)[TPT], double (&fxa)[TPT], double (&fya)[TPT],
                                          double (&fza)[TPT], double (&pta)[TPT], const int (&ia)[TPT],
                                          double (&xb)[SPT], double (&yb)[SPT], double (&zb)[SPT],
                                          double (&qb)[SPT], double (&fxb)[SPT], double (&fyb)[SPT],
                                          double (&fzb)[SPT], double (&ptb)[SPT], const int (&ib)[SPT], double eps2) {
#pragma unroll
  for (int v = 0; v < SPT; ++v) {
#pragma unroll
    for (int u = 0; u < TPT; ++u) {
      const double dx = xa[u] - xb[v], dy = ya[u] - yb[v], dz = za[u] - zb[v];
      const double r2 = fma(dx, dx, fma(dy, dy, fma(dz, dz, eps2)));
      double w = rsqrt_fast(r2);
      if (DIAG) w = ib[v] > ia[u] ? w : 0.0;
      const double pa_ = qa[u] * w, pb_ = qb[v] * w;
      const double s = pa_ * pb_ * w;
      pta[u] += pb_;
      ptb[v] += pa_;
      fxa[u] = fma(s, dx, fxa[u]);
      fya[u] = fma(s, dy, fya[u]);
      fza[u] = fma(s, dz, fza[u]);
      fxb[v] = fma(-s, dx, fxb[v]);
      fyb[v] = fma(-s, dy, fyb[v]);
      fzb[v] = fma(-s, dz, fzb[v]);
    }
  }
}

template <bool DIAG>
__device__ __forceinline__ void run_block(const P2PArgs& A, int ba, int bb, double (*red)[4][CHUNK]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double xa[TPT], ya[TPT], za[TPT], qa[TPT], fxa[TPT], fya[TPT], fza[TPT], pta[TPT];
  int ia[TPT];
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    ia[u] = ba * BLK + warp * (32 * TPT) + u * 32 + lane;
    const bool ok = ia[u] < A.na;
    const int t = ok ? ia[u] : 0;
    xa[u] = ok ? A.pa[t] : FAR;
    ya[u] = ok ? A.pa[A.ld_pa + t] : FAR;
    za[u] = ok ? A.pa[2 * A.ld_pa + t] : FAR;
    qa[u] = ok ? A.pa[3 * A.ld_pa + t] : 0.0;
    fxa[u] = fya[u] = fza[u] = pta[u] = 0.0;
  }
  const int b_end = min(A.nb, (bb + 1) * BLK);
  for (int c0 = bb * BLK; c0 < b_end; c0 += CHUNK) {
    double xb[SPT], yb[SPT], zb[SPT], qb[SPT], fxb[SPT], fyb[SPT], fzb[SPT], ptb[SPT];
    int ib[SPT];
#pragma unroll
    for (int v = 0; v < SPT; ++v) {
      ib[v] = c0 + v * 32 + lane;
      const bool ok = ib[v] < b_end;
      const int t = ok ? ib[v] : 0;
      xb[v] = ok ? A.pb[t] : -FAR;
      yb[v] = ok ? A.pb[A.ld_pb + t] : -FAR;
      zb[v] = ok ? A.pb[2 * A.ld_pb + t] : -FAR;
      qb[v] = ok ? A.pb[3 * A.ld_pb + t] : 0.0;
      fxb[v] = fyb[v] = fzb[v] = ptb[v] = 0.0;
    }
    const int src = (lane + 1) & 31;
#pragma unroll 1
    for (int r = 0; r < 32; ++r) {
      pair_step<DIAG>(xa, ya, za, qa, fxa, fya, fza, pta, ia, xb, yb, zb, qb, fxb, fyb, fzb, ptb, ib, A.eps2);
#pragma unroll
      for (int v = 0; v < SPT; ++v) {
        xb[v] = __shfl_sync(0xffffffffu, xb[v], src);
        yb[v] = __shfl_sync(0xffffffffu, yb[v], src);
        zb[v] = __shfl_sync(0xffffffffu, zb[v], src);
        qb[v] = __shfl_sync(0xffffffffu, qb[v], src);
        fxb[v] = __shfl_sync(0xffffffffu, fxb[v], src);
        fyb[v] = __shfl_sync(0xffffffffu, fyb[v], src);
        fzb[v] = __shfl_sync(0xffffffffu, fzb[v], src);
        ptb[v] = __shfl_sync(0xffffffffu, ptb[v], src);
        if (DIAG) ib[v] = __shfl_sync(0xffffffffu, ib[v], src);
      }
    }
    // 32 rotations: every source is home again.  Sum the 4 warps' partials.
#pragma unroll
    for (int v = 0; v < SPT; ++v) {
      red[warp][0][v * 32 + lane] = fxb[v];
      red[warp][1][v * 32 + lane] = fyb[v];
      red[warp][2][v * 32 + lane] = fzb[v];
      red[warp][3][v * 32 + lane] = ptb[v];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 4 * CHUNK; e += THREADS) {
      const int comp = e / CHUNK, k = e - comp * CHUNK;
      const int j = c0 + k;
      if (j < b_end) {
        const double sum = (red[0][comp][k] + red[1][comp][k]) + (red[2][comp][k] + red[3][comp][k]);
        atomicAdd(&A.fb[comp * A.ld_fb + j], sum);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const int t = ia[u];
    if (t >= A.na) continue;
    atomicAdd(&A.fa[t], fxa[u]);
    atomicAdd(&A.fa[A.ld_fa + t], fya[u]);
    atomicAdd(&A.fa[2 * A.ld_fa + t], fza[u]);
    atomicAdd(&A.fa[3 * A.ld_fa + t], pta[u]);
  }
}

// ---- deterministic one-sided evaluation (runtime option "deterministic") ----
// Every target is owned by ONE thread of ONE CTA, which walks all sources of the
// other side in a fixed order (staged through shared memory, broadcast reads)
// and finally adds its sums into F with a plain read-modify-write: no atomics,
// so the result is bitwise repeatable.  A pair task is two passes in one
// launch (CTAs for the targets of side i with sources j, then the reverse); it
// costs the one-directional 21 FP64 ops per ORDERED interaction instead of
// 11.5, the price of the fixed order.  The runtime runs commutative members
// one at a time in this mode (exclusive guards), so the plain update is safe.
constexpr int DET_THREADS = 256;
constexpr int DET_TPT = 2;  // targets per thread
constexpr int DET_BLK = DET_THREADS * DET_TPT;
constexpr int DET_CHUNK = 256;  // sources staged per round

struct DetArgs {
  const double* pt;  // targets: 4 x nt
  const double* ps;  // sources: 4 x ns
  double* ft;
  long long ld_pt, ld_ps, ld_ft;
  int nt, ns;
  int self;  // the source set is the target set: skip a == b
  double eps2;
};

__global__ void __launch_bounds__(DET_THREADS) p2p_det_kernel(DetArgs A0, DetArgs A1, int nblk0) {
  __shared__ double sx[DET_CHUNK], sy[DET_CHUNK], sz[DET_CHUNK], sq[DET_CHUNK];
  const bool second = static_cast<int>(blockIdx.x) >= nblk0;
  const DetArgs& A = second ? A1 : A0;
  const int blk = second ? blockIdx.x - nblk0 : blockIdx.x;
  double x[DET_TPT], y[DET_TPT], z[DET_TPT], q[DET_TPT], fx[DET_TPT], fy[DET_TPT], fz[DET_TPT], pt[DET_TPT];
  int ia[DET_TPT];
#pragma unroll
  for (int u = 0; u < DET_TPT; ++u) {
    ia[u] = blk * DET_BLK + u * DET_THREADS + threadIdx.x;
    const bool ok = ia[u] < A.nt;
    const int t = ok ? ia[u] : 0;
    x[u] = A.pt[t];
    y[u] = A.pt[A.ld_pt + t];
    z[u] = A.pt[2 * A.ld_pt + t];
    q[u] = A.pt[3 * A.ld_pt + t];
    fx[u] = fy[u] = fz[u] = pt[u] = 0.0;
  }
  for (int c0 = 0; c0 < A.ns; c0 += DET_CHUNK) {
    __syncthreads();
    for (int e = threadIdx.x; e < DET_CHUNK; e += DET_THREADS) {
      const int j = c0 + e;
      const bool ok = j < A.ns;
      sx[e] = ok ? A.ps[j] : FAR;
      sy[e] = ok ? A.ps[A.ld_ps + j] : FAR;
      sz[e] = ok ? A.ps[2 * A.ld_ps + j] : FAR;
      sq[e] = ok ? A.ps[3 * A.ld_ps + j] : 0.0;
    }
    __syncthreads();
    const int cn = min(DET_CHUNK, A.ns - c0);
    for (int e = 0; e < cn; ++e) {
      const double bx = sx[e], by = sy[e], bz = sz[e], bq = sq[e];
#pragma unroll
      for (int u = 0; u < DET_TPT; ++u) {
        const double dx = x[u] - bx, dy = y[u] - by, dz = z[u] - bz;
        const double r2 = fma(dx, dx, fma(dy, dy, fma(dz, dz, A.eps2)));
        double w = rsqrt_fast(r2);
        if (A.self && c0 + e == ia[u]) w = 0.0;
        const double pb = bq * w;
        const double s = q[u] * pb * w * w;
        pt[u] += pb;
        fx[u] = fma(s, dx, fx[u]);
        fy[u] = fma(s, dy, fy[u]);
        fz[u] = fma(s, dz, fz[u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < DET_TPT; ++u) {
    const int t = ia[u];
    if (t >= A.nt) continue;
    A.ft[t] += fx[u];
    A.ft[A.ld_ft + t] += fy[u];
    A.ft[2 * A.ld_ft + t] += fz[u];
    A.ft[3 * A.ld_ft + t] += pt[u];
  }
}

constexpr int MAX_GROUP = 32;

// One launch for up to MAX_GROUP tasks of the same op (grouped by the
// runtime's executor like the DGEMMs): task k owns CTAs [first[k], first[k+1]).
// Pair task: nblk_a * nblk_b CTAs; self task (SELF): the nblk (nblk + 1) / 2
// blocks ba <= bb of one group.
struct P2PGroup {
  P2PArgs t[MAX_GROUP];
  int first[MAX_GROUP + 1];
  int n;
};

template <bool SELF>
__global__ void __launch_bounds__(THREADS) p2p_mutual_kernel(const __grid_constant__ P2PGroup G) {
  __shared__ double red[THREADS / 32][4][CHUNK];
  int k = 0;
  while (k + 1 < G.n && static_cast<int>(blockIdx.x) >= G.first[k + 1]) ++k;
  const P2PArgs& A = G.t[k];
  int lin = blockIdx.x - G.first[k];
  int ba, bb;
  if (SELF) {
    ba = 0;
    while (lin >= A.nblk_a - ba) {
      lin -= A.nblk_a - ba;
      ++ba;
    }
    bb = ba + lin;
  } else {
    ba = lin / A.nblk_b;
    bb = lin - ba * A.nblk_b;
  }
  if (SELF && ba == bb)
    run_block<true>(A, ba, bb, red);
  else
    run_block<false>(A, ba, bb, red);
}

}  // namespace

cudaError_t launch_p2p_group(const P2PDesc* d, int ntasks, bool self, double eps2, cudaStream_t s) {
  for (int c0 = 0; c0 < ntasks; c0 += MAX_GROUP) {
    P2PGroup G{};
    G.n = 0;
    int blocks = 0;
    for (int k = c0; k < ntasks && k < c0 + MAX_GROUP; ++k) {
      const P2PDesc& x = d[k];
      if (x.ni <= 0 || (!self && x.nj <= 0)) continue;
      P2PArgs& a = G.t[G.n];
      a.pa = x.Pi;
      a.fa = x.Fi;
      a.ld_pa = x.ldpi;
      a.ld_fa = x.ldfi;
      a.na = x.ni;
      a.nblk_a = (x.ni + BLK - 1) / BLK;
      a.eps2 = eps2;
      if (self) {
        a.pb = x.Pi;
        a.fb = x.Fi;
        a.ld_pb = x.ldpi;
        a.ld_fb = x.ldfi;
        a.nb = x.ni;
        a.nblk_b = a.nblk_a;
      } else {
        a.pb = x.Pj;
        a.fb = x.Fj;
        a.ld_pb = x.ldpj;
        a.ld_fb = x.ldfj;
        a.nb = x.nj;
        a.nblk_b = (x.nj + BLK - 1) / BLK;
      }
      G.first[G.n] = blocks;
      blocks += self ? a.nblk_a * (a.nblk_a + 1) / 2 : a.nblk_a * a.nblk_b;
      ++G.n;
    }
    if (!G.n) continue;
    G.first[G.n] = blocks;
    count_launch();
    if (self)
      p2p_mutual_kernel<true><<<blocks, THREADS, 0, s>>>(G);
    else
      p2p_mutual_kernel<false><<<blocks, THREADS, 0, s>>>(G);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_p2p(const double* Pi, long long ldpi, int ni, const double* Pj, long long ldpj, int nj, double* Fi,
                       long long ldfi, double* Fj, long long ldfj, bool self, double eps2, cudaStream_t s) {
  if (deterministic_launches()) {
    if (ni <= 0 || (!self && nj <= 0)) return cudaSuccess;
    DetArgs a0{Pi, self ? Pi : Pj, Fi, ldpi, self ? ldpi : ldpj, ldfi, ni, self ? ni : nj, self ? 1 : 0, eps2};
    DetArgs a1 = a0;
    const int nb0 = (ni + DET_BLK - 1) / DET_BLK;
    int blocks = nb0;
    if (!self) {
      a1 = DetArgs{Pj, Pi, Fj, ldpj, ldpi, ldfj, nj, ni, 0, eps2};
      blocks += (nj + DET_BLK - 1) / DET_BLK;
    }
    count_launch();
    p2p_det_kernel<<<blocks, DET_THREADS, 0, s>>>(a0, a1, nb0);
    return cudaGetLastError();
  }
  P2PDesc d{Pi, ldpi, ni, Pj, ldpj, nj, Fi, ldfi, Fj, ldfj};
  return launch_p2p_group(&d, 1, self, eps2, s);
}

}  // namespace sfx
