// Small device ops: generators (bit-identical to oracle/inputs.py), the
// runtime's test ops (spin, int64 cell arithmetic, byte adds) and the FP64
// DMMA peak microbenchmark used as the roofline denominator.
#include "kernels.h"
#include "ptx.cuh"

namespace sfx {

std::atomic<unsigned long long> g_kernel_launches{0};

namespace {

constexpr long long kMod = 10000019;  // reference tests/conftest.py:22

__device__ __forceinline__ double splitmix_uniform(unsigned long long seed, unsigned long long g) {
  // oracle/inputs.py: z = seed*GOLDEN + g; splitmix64 finaliser; 53-bit mantissa
  unsigned long long z = seed * 0x9E3779B97F4A7C15ull + g;
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return static_cast<double>(z >> 11) * 0x1.0p-53;
}

__global__ void fill_uniform_kernel(double* a, long long rows, long long cols, long long ld, unsigned long long seed,
                                    long long row0, long long col0, long long ncols_total) {
  long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= rows * cols) return;
  long long r = i / cols, c = i % cols;
  unsigned long long g = static_cast<unsigned long long>(row0 + r) * ncols_total + (col0 + c);
  a[r * ld + c] = splitmix_uniform(seed, g);
}

__global__ void fill_spd_kernel(double* a, long long rows, long long cols, long long ld, unsigned long long seed,
                                long long row0, long long col0, long long n) {
  long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= rows * cols) return;
  long long r = i / cols, c = i % cols;
  long long I = row0 + r, J = col0 + c;
  double u1 = splitmix_uniform(seed, static_cast<unsigned long long>(I) * n + J);
  double u2 = splitmix_uniform(seed, static_cast<unsigned long long>(J) * n + I);
  double v = (u1 + u2) * 0.5;
  if (I == J) v += static_cast<double>(n);
  a[r * ld + c] = v;
}

__global__ void fill_particles_kernel(double* p, long long n, long long ld, unsigned long long seed, long long first) {
  long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  unsigned long long g = static_cast<unsigned long long>(first + i) * 4ull;
  p[0 * ld + i] = splitmix_uniform(seed, g + 0);
  p[1 * ld + i] = splitmix_uniform(seed, g + 1);
  p[2 * ld + i] = splitmix_uniform(seed, g + 2);
  p[3 * ld + i] = 0.5 + 0.5 * splitmix_uniform(seed, g + 3);
}

__global__ void spin_kernel(long long ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned long long t = t0;
  while (t - t0 < static_cast<unsigned long long>(ns)) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
}

__device__ __forceinline__ long long pymod(long long x) { return ((x % kMod) + kMod) % kMod; }

struct CellArgs {
  long long* target;
  const long long* reads[7];
  int nreads;
  long long kind, a, b;
};

__global__ void cell_kernel(CellArgs c) {
  long long rsum = 0;
  for (int k = 0; k < c.nreads; ++k) rsum += *c.reads[k];
  long long t = *c.target;
  switch (c.kind) {
    case 1:
      *c.target = pymod(c.a * t + c.b + rsum);
      break;
    case 2:
      if (t % 2 == 0) *c.target = pymod(c.a * t + c.b + rsum);
      break;
    case 3: {
      // members of an atomic slot run concurrently: the body brings its own atomicity
      long long contrib = pymod(c.b + rsum);
      unsigned long long* p = reinterpret_cast<unsigned long long*>(c.target);
      unsigned long long old = *p, assumed;
      do {
        assumed = old;
        long long nv = pymod(static_cast<long long>(assumed) + contrib);
        old = atomicCAS(p, assumed, static_cast<unsigned long long>(nv));
      } while (old != assumed);
      break;
    }
    case 4:
      *c.target = pymod(t + c.b + c.a * rsum);
      break;
    default:
      break;
  }
}

__global__ void bytes_add_kernel(unsigned char* p, long long off, long long len, long long delta) {
  long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= len) return;
  p[off + i] = static_cast<unsigned char>((static_cast<long long>(p[off + i]) + delta) & 255);
}

__global__ void dmma_peak_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) ptx::dmma_8x8x4(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// FP64 pipe (DFMA) peak: 8 independent FMA chains per thread
__global__ void dfma_peak_kernel(double* out, int iters) {
  double a = 1.0 - threadIdx.x * 1e-9, b = 1e-9 * blockIdx.x;
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

inline unsigned grid_for(long long n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

}  // namespace

cudaError_t launch_fill_uniform(double* a, long long rows, long long cols, long long ld, long long seed,
                                long long row0, long long col0, long long ncols_total, cudaStream_t s) {
  long long n = rows * cols;
  if (n <= 0) return cudaSuccess;
  count_launch();
  fill_uniform_kernel<<<grid_for(n, 256), 256, 0, s>>>(a, rows, cols, ld, seed, row0, col0, ncols_total);
  return cudaGetLastError();
}

cudaError_t launch_fill_spd(double* a, long long rows, long long cols, long long ld, long long seed, long long row0,
                            long long col0, long long n, cudaStream_t s) {
  long long m = rows * cols;
  if (m <= 0) return cudaSuccess;
  count_launch();
  fill_spd_kernel<<<grid_for(m, 256), 256, 0, s>>>(a, rows, cols, ld, seed, row0, col0, n);
  return cudaGetLastError();
}

cudaError_t launch_fill_particles(double* p, long long n, long long ld, long long seed, long long first,
                                  cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_launch();
  fill_particles_kernel<<<grid_for(n, 256), 256, 0, s>>>(p, n, ld, seed, first);
  return cudaGetLastError();
}

namespace {
struct AddI64Args {
  long long* cells[8];
  int n;
  long long delta;
};
// SFX_OP_ADD_I64: device-atomic accumulation (members of one commutative group
// may run concurrently, runtime.h accumulates_atomically)
__global__ void add_i64_kernel(AddI64Args a) {
  if (threadIdx.x < a.n)
    atomicAdd(reinterpret_cast<unsigned long long*>(a.cells[threadIdx.x]), static_cast<unsigned long long>(a.delta));
}
}  // namespace

namespace {
struct DaccArgs {
  double* a;
  const double* add[7];
  long long ld[7];
  long long lda, rows, cols;
  int n;
};
// SFX_OP_DACC: a += add_1 + ... + add_n, one element per thread (HBM-bound; the
// addends are per-GPU partial accumulators pulled peer-to-peer before the launch)
__global__ void dacc_kernel(DaccArgs p) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= p.rows * p.cols) return;
  const long long r = i / p.cols, c = i - r * p.cols;
  double v = p.a[r * p.lda + c];
  for (int k = 0; k < p.n; ++k) v += p.add[k][r * p.ld[k] + c];
  p.a[r * p.lda + c] = v;
}
}  // namespace

cudaError_t launch_dacc(double* a, long long lda, long long rows, long long cols, const double* const* add,
                        const long long* ld, int n, cudaStream_t s) {
  DaccArgs p{};
  p.a = a;
  p.lda = lda;
  p.rows = rows;
  p.cols = cols;
  p.n = n < 7 ? n : 7;
  for (int k = 0; k < p.n; ++k) {
    p.add[k] = add[k];
    p.ld[k] = ld[k];
  }
  if (rows * cols <= 0) return cudaSuccess;
  count_launch();
  dacc_kernel<<<grid_for(rows * cols, 256), 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_add_i64(long long* const* cells, int n, long long delta, cudaStream_t s) {
  AddI64Args a{};
  a.n = n < 8 ? n : 8;
  for (int k = 0; k < a.n; ++k) a.cells[k] = cells[k];
  a.delta = delta;
  count_launch();
  add_i64_kernel<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

__global__ void fault_kernel(int kind) {
  if (kind == 1) __trap();
}

cudaError_t launch_fault(int kind, cudaStream_t s) {
  count_launch();
  if (kind == 0)
    fault_kernel<<<1, 4096, 0, s>>>(0);  // > 1024 threads per block: cudaErrorInvalidConfiguration
  else
    fault_kernel<<<1, 32, 0, s>>>(1);
  return cudaGetLastError();
}

cudaError_t launch_spin(long long ns, cudaStream_t s) {
  count_launch();
  spin_kernel<<<1, 32, 0, s>>>(ns);
  return cudaGetLastError();
}

// n same-duration spin tasks of one launch group: one CTA each, all concurrent
// (the overhead protocol's bodies of n ready chains in one launch)
cudaError_t launch_spin_group(int n, long long ns, cudaStream_t s) {
  count_launch();
  spin_kernel<<<n, 32, 0, s>>>(ns);
  return cudaGetLastError();
}

cudaError_t launch_cell(long long* target, const long long* const* reads, int nreads, long long kind, long long a,
                        long long b, cudaStream_t s) {
  CellArgs c;
  c.target = target;
  c.nreads = nreads;
  for (int k = 0; k < nreads && k < 7; ++k) c.reads[k] = reads[k];
  c.kind = kind;
  c.a = a;
  c.b = b;
  count_launch();
  cell_kernel<<<1, 1, 0, s>>>(c);
  return cudaGetLastError();
}

cudaError_t launch_bytes_add(unsigned char* p, long long off, long long len, long long delta, cudaStream_t s) {
  if (len <= 0) return cudaSuccess;
  count_launch();
  bytes_add_kernel<<<grid_for(len, 256), 256, 0, s>>>(p, off, len, delta);
  return cudaGetLastError();
}

cudaError_t fp64_dfma_peak(int iters, double* tflops) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaError_t e = cudaMalloc(&out, 8);
  if (e) return e;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 512, blocks = 4 * sms;
  count_launch();
  dfma_peak_kernel<<<blocks, threads>>>(out, 100);  // warm-up
  cudaEventRecord(e0);
  count_launch();
  dfma_peak_kernel<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  e = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  *tflops = 2.0 * 8 * static_cast<double>(iters) * blocks * threads / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return e ? e : cudaGetLastError();
}

cudaError_t fp64_dmma_peak(int iters, double* tflops) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaError_t e = cudaMalloc(&out, 8);
  if (e) return e;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int warps = 16;
  count_launch();
  dmma_peak_kernel<<<sms, 32 * warps>>>(out, 100);  // warm-up
  cudaEventRecord(e0);
  count_launch();
  dmma_peak_kernel<<<sms, 32 * warps>>>(out, iters);
  cudaEventRecord(e1);
  e = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  *tflops = 2.0 * 256 * 8 * static_cast<double>(iters) * sms * warps / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return e ? e : cudaGetLastError();
}

}  // namespace sfx
