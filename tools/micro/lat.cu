// Latency microbenchmarks for the POTRF pivot chain (clock64 deltas, one CTA)
#include <cstdio>
__global__ void k(double* out, long long* cyc, double seed) {
  __shared__ double sh[64];
  const int tid = threadIdx.x;
  double x = seed + tid * 1e-9;
  long long t0, t1;
  // 1. dependent DFMA chain
  __syncthreads();
  t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64();
  if (tid == 0) cyc[0] = (t1 - t0);
  // 2. dependent DMUL chain
  __syncthreads();
  t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = x * 1.0000001;
  t1 = clock64();
  if (tid == 0) cyc[1] = (t1 - t0);
  // 3. rsqrt.approx.f64 chain
  __syncthreads();
  t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; ++i) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y + 1.0; }
  t1 = clock64();
  if (tid == 0) cyc[2] = (t1 - t0);
  // 4. barrier alone (all warps)
  __syncthreads();
  t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; ++i) __syncthreads();
  t1 = clock64();
  if (tid == 0) cyc[3] = (t1 - t0);
  // 5. STS by one thread -> barrier -> LDS by all -> dependent use
  __syncthreads();
  t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; ++i) {
    if (tid == (i & 255)) sh[i & 63] = x;
    __syncthreads();
    x = sh[i & 63] + 1.0;
  }
  t1 = clock64();
  if (tid == 0) cyc[4] = (t1 - t0);
  // 6. full pivot-like chain: STS -> BAR -> LDS -> rsqrt+2 Newton -> DMUL -> DFMA
  __syncthreads();
  t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; ++i) {
    if (tid == (i & 255)) sh[i & 63] = x;
    __syncthreads();
    double d = sh[i & 63] + 2.0;
    double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    const double h = 0.5 * d;
    y = y * fma(-h * y, y, 1.5);
    y = y * fma(-h * y, y, 1.5);
    x = fma(-(d * y), y, x) * 0.5;
  }
  t1 = clock64();
  if (tid == 0) cyc[5] = (t1 - t0);
  out[tid] = x;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096 * 8); cudaMallocManaged(&cyc, 64 * 8);
  for (int threads : {32, 256}) {
    k<<<1, threads>>>(out, cyc, 1.0); cudaDeviceSynchronize();
    k<<<1, threads>>>(out, cyc, 1.0); cudaDeviceSynchronize();
    printf("threads %d: DFMA %.1f  DMUL %.1f  RSQ64 %.1f  BAR %.1f  STS-BAR-LDS-DADD %.1f  pivot-chain %.1f cyc/iter\n", threads,
           cyc[0] / 1000.0, cyc[1] / 1000.0, cyc[2] / 1000.0, cyc[3] / 1000.0, cyc[4] / 1000.0, cyc[5] / 1000.0);
  }
  return 0;
}
