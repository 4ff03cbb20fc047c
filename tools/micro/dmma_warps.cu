// DMMA.8x8x4 throughput vs warps per SM and independent accumulators per warp
#include <cstdio>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int ACC>
__global__ void k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
template <int ACC>
void run(int warps, double* out) {
  int sms = 148; cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096 * 8 / ACC;
  k<ACC><<<sms, 32 * warps>>>(out, 10);
  cudaEventRecord(e0); k<ACC><<<sms, 32 * warps>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("warps/SM %2d acc %2d: %.2f TFLOP/s\n", warps, ACC, 2.0 * 256 * ACC * (double)iters * sms * warps / (ms * 1e-3) / 1e12);
}
int main() {
  double* out; cudaMalloc(&out, 8);
  for (int w : {4, 8, 12, 16}) { run<8>(w, out); run<32>(w, out); }
}
