// FP64 issue cost per SMSP: N independent DFMA per thread per iteration, 8 warps
#include <cstdio>
template <int N>
__global__ void k(double* out, long long* cyc) {
  double a[32];
  for (int i = 0; i < 32; ++i) a[i] = threadIdx.x + i;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 1000; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) a[i] = fma(a[i], 0.9999999, 1e-9);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[N] = t1 - t0;
  double s = 0;
  for (int i = 0; i < 32; ++i) s += a[i];
  out[threadIdx.x] = s;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096 * 8); cudaMallocManaged(&cyc, 64 * 8);
  for (int th : {32, 128, 256}) {
    for (int rep = 0; rep < 2; ++rep) {
      k<1><<<1, th>>>(out, cyc); k<4><<<1, th>>>(out, cyc); k<8><<<1, th>>>(out, cyc); k<16><<<1, th>>>(out, cyc); k<32><<<1, th>>>(out, cyc);
      cudaDeviceSynchronize();
    }
    printf("threads %d: cyc/iter N=1 %.1f N=4 %.1f N=8 %.1f N=16 %.1f N=32 %.1f\n", th, cyc[1] / 1e3, cyc[4] / 1e3, cyc[8] / 1e3, cyc[16] / 1e3, cyc[32] / 1e3);
  }
}
