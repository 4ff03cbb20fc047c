// extern "C" entry points declared in include/sfx.h.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "kernels/kernels.h"
#include "runtime/runtime.h"

struct sfx_runtime {
  sfx::Runtime* rt;
};

namespace {
thread_local std::string g_err;

template <class F>
int guarded(sfx_runtime* r, F&& f) {
  if (!r || !r->rt) {
    g_err = "null runtime";
    return SFX_ERR_CONFIG;
  }
  try {
    return f(*r->rt);
  } catch (const std::bad_alloc&) {
    r->rt->last_error = "host out of memory";
    return SFX_ERR_INTERNAL;
  } catch (const std::exception& e) {
    r->rt->last_error = e.what();
    return SFX_ERR_INTERNAL;
  }
}
}  // namespace

extern "C" {

int sfx_abi_version(void) { return SFX_ABI_VERSION; }

int sfx_device_count(int* n) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  *n = c;
  return SFX_OK;
}

int sfx_create(int ndev, const int* ordinals, int streams_per_dev, const uint64_t* arena_bytes, uint32_t sched,
               uint32_t flags, uint32_t window, sfx_runtime** out) {
  *out = nullptr;
  if (ndev <= 0 || ndev > 64 || streams_per_dev <= 0 || streams_per_dev > 64) {
    g_err = "need 1..64 devices and 1..64 streams per device";
    return SFX_ERR_CONFIG;
  }
  if (sched != SFX_SCHED_FIFO && sched != SFX_SCHED_PRIO) {
    g_err = "unknown scheduler";
    return SFX_ERR_CONFIG;
  }
  const bool sim = flags & SFX_FLAG_SIM;
  if (!sim) {
    int have = 0;
    sfx_device_count(&have);
    for (int d = 0; d < ndev; ++d) {
      int ord = ordinals ? ordinals[d] : d;
      if (ord < 0 || ord >= have) {
        g_err = "CUDA device " + std::to_string(ord) + " is not available (" + std::to_string(have) +
                " visible); the GPU engine has no CPU fallback";
        return SFX_ERR_CUDA;
      }
    }
  }
  // arena allocation granularity: bits 8..15 of flags = log2(align), 0 = default
  uint32_t lg = (flags >> 8) & 0xff;
  uint64_t align = lg ? (1ull << lg) : (sim ? 8 : 256);
  sfx::Backend* be = sim ? sfx::make_sim_backend(ndev) : sfx::make_cuda_backend(ndev, ordinals, flags & SFX_FLAG_TRACE);
  auto* rt = new sfx::Runtime(be, ndev, streams_per_dev, sched, flags, window, align);
  std::string err;
  int rc = rt->init(arena_bytes, err);
  if (rc) {
    g_err = err;
    delete rt;
    return rc;
  }
  *out = new sfx_runtime{rt};
  return SFX_OK;
}

int sfx_destroy(sfx_runtime* r) {
  if (!r) return SFX_OK;
  delete r->rt;
  delete r;
  return SFX_OK;
}

const char* sfx_last_error(sfx_runtime* r) {
  if (!r || !r->rt) return g_err.c_str();
  return r->rt->last_error.c_str();
}

int sfx_failure(sfx_runtime* r, int* code, char* msg, uint64_t cap) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.failure(code, msg, cap); });
}

int sfx_graph_create(sfx_runtime* r, uint32_t* gid) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.graph_create(gid); });
}

int sfx_register(sfx_runtime* r, uint32_t gid, uint64_t hid, void* host, uint64_t bytes, int64_t rows, int64_t cols,
                 int64_t ld, int32_t dtype) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.reg(gid, hid, host, bytes, rows, cols, ld, dtype); });
}

int sfx_set_home(sfx_runtime* r, uint64_t hid, int32_t device) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.set_home(hid, device); });
}

int sfx_unregister(sfx_runtime* r, uint64_t hid) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.unreg(hid); });
}

int sfx_submit(sfx_runtime* r, uint32_t n, const sfx_task_desc* tasks, const sfx_access* accesses) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.submit(n, tasks, accesses); });
}

int sfx_pause(sfx_runtime* r) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.pause(true); });
}

int sfx_resume(sfx_runtime* r) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.pause(false); });
}

int sfx_wait_all(sfx_runtime* r, uint32_t gid, double timeout_s) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.wait_all(gid, timeout_s); });
}

int sfx_wait_task(sfx_runtime* r, uint64_t tid, double timeout_s) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.wait_task(tid, timeout_s); });
}

int sfx_task_state(sfx_runtime* r, uint64_t tid, int32_t* state) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.task_state(tid, state); });
}

int sfx_flush(sfx_runtime* r, uint32_t gid, uint64_t tid, uint64_t hid, int32_t write_mode) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.flush(gid, tid, hid, write_mode); });
}

int sfx_stats(sfx_runtime* r, int dev, sfx_dev_stats* out) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.stats(dev, out); });
}

int sfx_extern_poll(sfx_runtime* r, uint64_t* tids, uint64_t cap, uint64_t* n, double timeout_s) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.extern_poll(tids, cap, n, timeout_s); });
}

int sfx_extern_done(sfx_runtime* r, uint64_t tid, int status, const char* msg) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.extern_done(tid, status, msg); });
}

int sfx_graph_option(sfx_runtime* r, uint32_t gid, const char* key, int64_t value) {
  if (!key) return SFX_ERR_CONFIG;
  return guarded(r, [&](sfx::Runtime& rt) { return rt.graph_option(gid, key, value); });
}

int sfx_live(sfx_runtime* r, uint64_t* tasks, uint64_t* slots, uint64_t* retired) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.live(tasks, slots, retired); });
}

int sfx_fail(sfx_runtime* r, const char* msg) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.fail(msg ? msg : "external agent failed"); });
}

int sfx_resident(sfx_runtime* r, int dev, uint64_t* hids, uint64_t cap, uint64_t* n) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.resident(dev, hids, cap, n); });
}

int sfx_block_state(sfx_runtime* r, uint64_t hid, int32_t dev, int32_t* state, int32_t* host_valid) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.block_state(hid, dev, state, host_valid); });
}

int sfx_trace(sfx_runtime* r, uint32_t gid, sfx_event* buf, uint64_t cap, uint64_t* n) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.trace(gid, buf, cap, n); });
}

int sfx_edges(sfx_runtime* r, uint32_t gid, uint64_t* src, uint64_t* dst, uint64_t* hid, uint64_t cap,
              uint64_t* n) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.edges(gid, src, dst, hid, cap, n); });
}

int sfx_violations(sfx_runtime* r, uint64_t* n) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.violations(n); });
}

int sfx_register_op(const char* name, sfx_user_launch_fn fn, void* user, uint32_t* op) {
  if (!op) {
    g_err = "sfx_register_op: null op out-pointer";
    return SFX_ERR_CONFIG;
  }
  std::string err;
  const int rc = sfx::register_user_op(name, fn, user, op, err);
  if (rc) g_err = err;
  return rc;
}

int sfx_set_option(sfx_runtime* r, const char* key, int64_t value) {
  return guarded(r, [&](sfx::Runtime& rt) { return rt.set_option(key ? key : "", value); });
}

int sfx_host_alloc(uint64_t bytes, int sim, void** out) {
  *out = nullptr;
  if (!bytes) bytes = 1;
  if (sim) {
    *out = aligned_alloc(4096, (bytes + 4095) / 4096 * 4096);
    if (!*out) {
      g_err = "host allocation failed";
      return SFX_ERR_INTERNAL;
    }
    return SFX_OK;
  }
  cudaError_t e = cudaHostAlloc(out, bytes, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    g_err = std::string("cudaHostAlloc: ") + cudaGetErrorString(e);
    cudaGetLastError();
    return SFX_ERR_CUDA;
  }
  return SFX_OK;
}

int sfx_host_free(void* p, int sim) {
  if (!p) return SFX_OK;
  if (sim) {
    free(p);
    return SFX_OK;
  }
  return cudaFreeHost(p) == cudaSuccess ? SFX_OK : SFX_ERR_CUDA;
}

int sfx_fp64_peak(int ordinal, double* tflops, double* sm_mhz) {
  int have = 0;
  sfx_device_count(&have);
  if (ordinal < 0 || ordinal >= have) {
    g_err = "no such CUDA device";
    return SFX_ERR_CUDA;
  }
  cudaSetDevice(ordinal);
  cudaError_t e = sfx::fp64_dmma_peak(20000, tflops);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, ordinal);
  if (sm_mhz) *sm_mhz = clk / 1000.0;
  if (e != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return SFX_ERR_CUDA;
  }
  return SFX_OK;
}

int sfx_fp64_dfma_peak(int ordinal, double* tflops) {
  int have = 0;
  sfx_device_count(&have);
  if (ordinal < 0 || ordinal >= have) {
    g_err = "no such CUDA device";
    return SFX_ERR_CUDA;
  }
  cudaSetDevice(ordinal);
  cudaError_t e = sfx::fp64_dfma_peak(20000, tflops);
  if (e != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return SFX_ERR_CUDA;
  }
  return SFX_OK;
}

int sfx_gemm_paths(uint64_t* out, uint32_t n) {
  if (!out) return SFX_ERR_CONFIG;
  for (uint32_t k = 0; k < n && k < SFX_GEMM_PATHS; ++k) out[k] = sfx::g_gemm_paths[k].load();
  return SFX_OK;
}

}  // extern "C"
