// Particle-group P2P interaction kernel (FP64, sm_100a).
//
// Blocks are 4 x n SoA tiles: positions P = (x, y, z, q), accumulators
// F = (fx, fy, fz, pot).  For target a and source b (a != b):
//   r2   = |x_a - x_b|^2 + eps2
//   pot_a += q_b / r
//   F_a  += q_a q_b (x_a - x_b) / r^3
// A pair task (i, j) evaluates both directions (targets in i from sources in
// j, and targets in j from sources in i) in one launch: every ORDERED
// interaction is evaluated exactly once, which is the unit of the metric
// (N(N-1) ordered interactions, 20 flop each by convention).
// The self task (i, i) skips a == b.
//
// Layout/roofline choices: one thread owns TPT targets in registers; source
// tiles are staged in shared memory with coalesced loads and read back as
// broadcasts (every lane reads the same source), so the inner loop is pure
// FP64 pipe work: 3 DADD + 3 DFMA (r2) + MUFU.RSQ64H + 8 (Newton) + 3 DMUL +
// 1 DADD + 3 DFMA = 21 FP64 ops per ordered interaction.
// Commutative accumulation into F is exclusive per handle (the runtime chains
// members of a commutative group), so the epilogue is a plain read-add-write.
//
// Oracle: oracle/bodies.py p2p_pair / p2p_self.
#include "kernels.h"

namespace sfx {
namespace {

constexpr int THREADS = 128;
constexpr int TPT = 2;     // targets per thread (ILP + one smem broadcast per 2 interactions)
constexpr int TILE = 256;  // sources staged per shared-memory round
constexpr int SPLIT_SRC = 1024;  // sources per block: a task spreads over (targets/256) x (sources/1024) blocks

// 1/sqrt(x) for normal x > 0 (r2 >= eps2 > 0 here): the MUFU.RSQ64H seed
// (~23 bits) refined by two Newton steps (~46 -> full double).  4 FP64 ops per
// step, no special-case slow path (CUDA's rsqrt(double) branches to one).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x * y, y, 1.0);
  y = fma(0.5 * y, e, y);
  e = fma(-x * y, y, 1.0);
  y = fma(0.5 * y, e, y);
  return y;
}

struct P2PSide {
  const double* tgt;  // 4 x nt (ld)
  const double* src;  // 4 x ns (ld)
  double* acc;        // 4 x nt (ld)
  long long ld_t, ld_s, ld_a;
  int nt, ns;
  int self;  // exclude a == b
};

__global__ void __launch_bounds__(THREADS) p2p_kernel(P2PSide s0, P2PSide s1, int blocks0, double eps2) {
  __shared__ double4 sp[TILE];
  const bool second = blockIdx.x >= blocks0;
  const P2PSide& S = second ? s1 : s0;
  const int blk_lin = second ? blockIdx.x - blocks0 : blockIdx.x;
  const int nsplit = (S.ns + SPLIT_SRC - 1) / SPLIT_SRC;
  const int blk = blk_lin / nsplit, split = blk_lin - blk * nsplit;
  const int j_begin = split * SPLIT_SRC, j_end = min(S.ns, j_begin + SPLIT_SRC);
  const int base = blk * THREADS * TPT;
  double xi[TPT], yi[TPT], zi[TPT];
  double ax[TPT], ay[TPT], az[TPT], ap[TPT];
  int ti[TPT];
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    ti[u] = base + u * THREADS + threadIdx.x;
    const int t = ti[u] < S.nt ? ti[u] : 0;
    xi[u] = S.tgt[t];
    yi[u] = S.tgt[S.ld_t + t];
    zi[u] = S.tgt[2 * S.ld_t + t];
    ax[u] = ay[u] = az[u] = ap[u] = 0.0;
  }
  for (int j0 = j_begin; j0 < j_end; j0 += TILE) {
    __syncthreads();
    for (int k = threadIdx.x; k < TILE; k += THREADS) {
      const int j = j0 + k;
      double4 v;
      if (j < j_end) {
        v.x = S.src[j];
        v.y = S.src[S.ld_s + j];
        v.z = S.src[2 * S.ld_s + j];
        v.w = S.src[3 * S.ld_s + j];
      } else {
        v.x = v.y = v.z = 0.0;
        v.w = 0.0;  // zero charge: contributes nothing
      }
      sp[k] = v;
    }
    __syncthreads();
    const int jn = min(TILE, j_end - j0);
#pragma unroll 4
    for (int k = 0; k < jn; ++k) {
      const double4 p = sp[k];
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        const double dx = xi[u] - p.x, dy = yi[u] - p.y, dz = zi[u] - p.z;
        const double r2 = fma(dx, dx, fma(dy, dy, fma(dz, dz, eps2)));
        double inv = rsqrt_nr(r2);
        if (S.self && j0 + k == ti[u]) inv = 0.0;
        const double qi = p.w * inv;        // q_b / r
        const double s3 = qi * inv * inv;   // q_b / r^3
        ap[u] += qi;
        ax[u] = fma(s3, dx, ax[u]);
        ay[u] = fma(s3, dy, ay[u]);
        az[u] = fma(s3, dz, az[u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const int t = ti[u];
    if (t >= S.nt) continue;
    // source splits of one task add into the same targets: FP64 atomics
    // (the runtime already keeps different tasks of a commutative group apart)
    const double qa = S.tgt[3 * S.ld_t + t];
    atomicAdd(&S.acc[t], qa * ax[u]);
    atomicAdd(&S.acc[S.ld_a + t], qa * ay[u]);
    atomicAdd(&S.acc[2 * S.ld_a + t], qa * az[u]);
    atomicAdd(&S.acc[3 * S.ld_a + t], ap[u]);
  }
}

}  // namespace

cudaError_t launch_p2p(const double* Pi, long long ldpi, int ni, const double* Pj, long long ldpj, int nj, double* Fi,
                       long long ldfi, double* Fj, long long ldfj, bool self, double eps2, cudaStream_t s) {
  const int per_block = THREADS * TPT;
  P2PSide a{Pi, self ? Pi : Pj, Fi, ldpi, self ? ldpi : ldpj, ldfi, ni, self ? ni : nj, self ? 1 : 0};
  const int b0 = (ni + per_block - 1) / per_block * ((a.ns + SPLIT_SRC - 1) / SPLIT_SRC);
  if (self) {
    count_launch();
    p2p_kernel<<<b0, THREADS, 0, s>>>(a, a, b0, eps2);
  } else {
    P2PSide b{Pj, Pi, Fj, ldpj, ldpi, ldfj, nj, ni, 0};
    const int b1 = (nj + per_block - 1) / per_block * ((b.ns + SPLIT_SRC - 1) / SPLIT_SRC);
    count_launch();
    p2p_kernel<<<b0 + b1, THREADS, 0, s>>>(a, b, b0, eps2);
  }
  return cudaGetLastError();
}

}  // namespace sfx
