// Pattern microbenchmark of one F pivot step: 8 warps, barrier, shared loads of
// the pivot column, one FP64 dependency chain, a published value (clock64 / iter)
#include <cstdio>
template <int MODE>
__global__ void k(double* out, long long* cyc) {
  __shared__ __align__(16) double col[2][64];
  const int tid = threadIdx.x, P = (tid >> 4) & 15, Q = tid & 15;
  double a[4] = {1.0 + tid, 2.0, 3.0, 4.0};
  if (tid < 128) (&col[0][0])[tid] = 1.0 + tid * 1e-3;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int j = 0; j < 64; ++j) {
    const int buf = j & 1;
    __syncthreads();
    const double d = col[buf][j];
    double2 c0 = *reinterpret_cast<const double2*>(&col[buf][4 * P]);
    double2 c1 = *reinterpret_cast<const double2*>(&col[buf][4 * Q]);
    double r = d;
    if (MODE >= 1) {  // 1/d chain
      double y;
      asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
      const double e = fma(-d, y, 1.0);
      const double t = fma(e, e, e);
      r = fma(y, t, y);
    }
    a[0] = fma(-(c0.x * c1.x), r, a[0]);
    a[1] = fma(-(c0.y * c1.x), r, a[1]);
    if (MODE >= 2) {
      a[2] = fma(-(c0.x * c1.y), r, a[2]);
      a[3] = fma(-(c0.y * c1.y), r, a[3]);
    }
    if (Q == ((j + 1) >> 2)) {
      col[buf ^ 1][4 * P] = a[0];
      col[buf ^ 1][4 * P + 1] = a[1];
    }
  }
  long long t1 = clock64();
  if (tid == 0) cyc[MODE] = t1 - t0;
  out[tid] = a[0] + a[1] + a[2] + a[3];
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096 * 8); cudaMallocManaged(&cyc, 64 * 8);
  for (int th : {128, 256}) {
    k<0><<<1, th>>>(out, cyc); k<1><<<1, th>>>(out, cyc); k<2><<<1, th>>>(out, cyc); cudaDeviceSynchronize();
    k<0><<<1, th>>>(out, cyc); k<1><<<1, th>>>(out, cyc); k<2><<<1, th>>>(out, cyc); cudaDeviceSynchronize();
    printf("threads %d: no-rcp %.1f  rcp %.1f  rcp+2 more fma %.1f cyc/pivot\n", th, cyc[0] / 64.0, cyc[1] / 64.0, cyc[2] / 64.0);
  }
}
