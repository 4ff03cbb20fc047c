// Example user op (sfx_register_op): Y += alpha * X on FP64 tiles.
//
// The reference runs any `device=` callable on the task's DeviceViews
// (src/engine.py:144-149, views from src/device.py:119-133).  On the B200 path a
// user op is a native LAUNCHER with the same information: the staged operands
// in declaration order (X read, Y write), the stream the runtime issues the task
// on, and the task's scalar parameters (fparam[0] = alpha).  It enqueues its
// kernel and returns; the runtime records the task's end event after it and
// releases successors from that event like for a built-in op.  On the
// simulated backend (stream == NULL) the views are host memory and the launcher
// computes on the host.
//
// Built by paper_2308_15964_b200/build.py into libsfx_user_daxpy.so; registered
// with paper_2308_15964_b200.ops.register("daxpy", <this symbol>).
#include <cuda_runtime.h>

#include "sfx.h"

namespace {

__global__ void __launch_bounds__(256) daxpy_tile(const double* __restrict__ x, long long ldx, double* __restrict__ y,
                                                  long long ldy, long long rows, long long cols, double alpha) {
  // one warp-strided row segment per thread block row: consecutive lanes hit
  // consecutive columns (coalesced 256-byte transactions per warp)
  for (long long r = blockIdx.y; r < rows; r += gridDim.y)
    for (long long c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += static_cast<long long>(gridDim.x) * blockDim.x)
      y[r * ldy + c] += alpha * x[r * ldx + c];
}

}  // namespace

extern "C" int sfx_example_daxpy(const sfx_view* v, int n, void* stream, const double* fparam, const int64_t*,
                                 void*) {
  if (n != 2 || v[0].dtype != SFX_DTYPE_F64 || v[1].dtype != SFX_DTYPE_F64 || v[0].rows != v[1].rows ||
      v[0].cols != v[1].cols)
    return 1;  // the runtime poisons the engine (SFX_ERR_USER)
  const double alpha = fparam[0];
  const double* x = static_cast<const double*>(v[0].data);
  double* y = static_cast<double*>(v[1].data);
  if (!stream) {  // simulated backend: host memory, synchronous
    for (int64_t r = 0; r < v[1].rows; ++r)
      for (int64_t c = 0; c < v[1].cols; ++c) y[r * v[1].ld + c] += alpha * x[r * v[0].ld + c];
    return 0;
  }
  const unsigned gx = static_cast<unsigned>((v[1].cols + 255) / 256);
  const unsigned gy = static_cast<unsigned>(v[1].rows < 1184 ? v[1].rows : 1184);  // 8 x 148 SMs
  if (!gx || !gy) return 0;
  daxpy_tile<<<dim3(gx, gy), 256, 0, static_cast<cudaStream_t>(stream)>>>(x, v[0].ld, y, v[1].ld, v[1].rows,
                                                                           v[1].cols, alpha);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}
