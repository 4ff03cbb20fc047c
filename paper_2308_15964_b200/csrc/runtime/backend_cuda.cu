// CUDA backend: one arena (single cudaMalloc slab) per device, K streams per
// device, pooled events, async H2D/D2H copies and cudaMemcpyPeerAsync over
// NVLink, and the op dispatch to the sm_100a kernels.
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>

#include "../kernels/kernels.h"
#include "runtime.h"

namespace sfx {
namespace {

inline int cuda_err(cudaError_t e, const char* what, std::string& err) {
  if (e == cudaSuccess) return SFX_OK;
  err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return SFX_ERR_CUDA;
}

struct Ev {
  cudaEvent_t e = nullptr;
  bool timing = false;
};
inline cudaEvent_t ev_of(void* p) { return static_cast<Ev*>(p)->e; }

class CudaBackend : public Backend {
  struct Dev {
    int ordinal = 0;
    std::vector<cudaStream_t> streams;
    char* arena = nullptr;
    uint64_t cap = 0;
    std::mutex pool_mu;
    std::vector<Ev*> pool_timing, pool_plain;
    cudaEvent_t base = nullptr;
    int64_t base_ns = 0;
    bool base_shared = false;  // base event owned by an earlier logical device on the same GPU
    // status words (DPOTRF info) in mapped pinned host memory: kernels store into
    // them directly, the completion thread reads them after the end event
    int* status = nullptr;
    int* status_dev = nullptr;
    std::vector<int> status_free;
    bool ready = false;
    std::vector<void*> scratch;  // per stream (cooperative streams only)
    // per stream, allocated on first use (stream-ordered): TRSM with the full
    // inverse computes X = B W^T out of place before copying it back
    std::vector<void*> tscratch;
    std::vector<size_t> tscratch_bytes;
  };

  void* trsm_scratch(int d, int stream, size_t need) {
    Dev& D = *devs_[d];
    if (D.tscratch.size() < D.streams.size()) {
      D.tscratch.resize(D.streams.size(), nullptr);
      D.tscratch_bytes.resize(D.streams.size(), 0);
    }
    if (D.tscratch_bytes[stream] < need) {
      // grow to the next power of two (a grouped TRSM launch needs one tile per
      // member, so sizes vary from launch to launch); the allocations come from
      // the device pool that init_device pre-backs and that keeps freed memory
      // (with the default release threshold, pool growth went back to the driver
      // on the executor's path: C3 factorizations took up to 2.7x longer at random)
      size_t want = size_t(1) << 20;
      while (want < need) want <<= 1;
      need = want;
      if (D.tscratch[stream]) cudaFreeAsync(D.tscratch[stream], D.streams[stream]);
      D.tscratch[stream] = nullptr;
      D.tscratch_bytes[stream] = 0;
      if (cudaMallocAsync(&D.tscratch[stream], need, D.streams[stream]) != cudaSuccess) {
        cudaGetLastError();
        D.tscratch[stream] = nullptr;
        return nullptr;
      }
      D.tscratch_bytes[stream] = need;
    }
    return D.tscratch[stream];
  }
  static constexpr size_t kScratchBytes = 64ull << 20;  // >= fullinv_workspace_bytes(2048) = 42 MiB
  static constexpr int kStatusSlots = 4096;
  int* status_ptr(int d, int slot) { return slot >= 0 ? devs_[d]->status_dev + slot : nullptr; }

 public:
  CudaBackend(int ndev, const int* ordinals) : devs_(ndev) {
    for (int d = 0; d < ndev; ++d) {
      devs_[d] = new Dev();
      devs_[d]->ordinal = ordinals ? ordinals[d] : d;
    }
  }
  ~CudaBackend() override {
    shutdown();
    for (Dev* d : devs_) delete d;
  }
  bool is_sim() const override { return false; }

  int init_device(int d, int, int nstreams, int nurgent, int ncoop, int nprefetch, uint64_t bytes,
                  std::string& err) override {
    Dev& D = *devs_[d];
    cudaError_t e = cudaSetDevice(D.ordinal);
    if (e) return cuda_err(e, "cudaSetDevice", err);
    cudaSetDeviceFlags(cudaDeviceScheduleYield);  // fails harmlessly if a context exists
    cudaGetLastError();
    e = cudaFree(nullptr);
    if (e) return cuda_err(e, "context init", err);
    if (!bytes) {
      size_t fr = 0, tot = 0;
      e = cudaMemGetInfo(&fr, &tot);
      if (e) return cuda_err(e, "cudaMemGetInfo", err);
      const uint64_t reserve = 10ull << 30;  // incl. the scratch pool backed below
      bytes = fr > 2 * reserve ? fr - reserve : fr / 2;
    }
    bytes = (bytes + 255) / 256 * 256;
    e = cudaMalloc(&D.arena, bytes);
    if (e) return cuda_err(e, "arena cudaMalloc", err);
    {
      // stream-ordered scratch (trsm_scratch) stays in the device's default pool
      // once freed instead of returning to the driver at every synchronisation
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, D.ordinal) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        // and back it now: the grouped TRSMs' per-stream scratch otherwise grows
        // the pool from the driver on the executor's path (the first C3
        // factorization of a run took 385-815 ms instead of 366).  6 GiB: every
        // stream of a device can hold a launch group of b = 1024 tiles (~42
        // streams x 64 MiB); with 2 GiB, streams that met their first big TRSM
        // group late still grew the pool mid-run (C3 reps of 390-580 ms among
        // 356 ms ones, tools/r4k_var.sh).  The pool is per physical GPU, so
        // logical devices sharing one reuse the same backing.
        void* warm = nullptr;
        if (cudaMallocAsync(&warm, size_t(6) << 30, 0) == cudaSuccess ||
            (cudaGetLastError(), cudaMallocAsync(&warm, size_t(2) << 30, 0) == cudaSuccess)) {
          cudaFreeAsync(warm, 0);
          cudaStreamSynchronize(0);
        }
      }
      cudaGetLastError();
    }
    D.cap = bytes;
    e = cudaHostAlloc(reinterpret_cast<void**>(&D.status), kStatusSlots * sizeof(int),
                      cudaHostAllocMapped | cudaHostAllocPortable);
    if (e) return cuda_err(e, "cudaHostAlloc status words", err);
    memset(D.status, 0, kStatusSlots * sizeof(int));
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&D.status_dev), D.status, 0);
    if (e) return cuda_err(e, "cudaHostGetDevicePointer", err);
    D.status_free.clear();
    for (int k = kStatusSlots; k-- > 0;) D.status_free.push_back(k);
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    const int total = nstreams + nurgent + ncoop + nprefetch;
    D.streams.resize(total);
    D.scratch.assign(total, nullptr);
    for (int s = 0; s < total; ++s) {
      e = cudaStreamCreateWithPriority(&D.streams[s], cudaStreamNonBlocking, s < nstreams ? least : greatest);
      if (e) return cuda_err(e, "cudaStreamCreate", err);
      if (s >= nstreams + nurgent && s < nstreams + nurgent + ncoop) {  // cooperative-kernel streams
        e = cudaMalloc(&D.scratch[s], kScratchBytes);
        if (e) return cuda_err(e, "scratch cudaMalloc", err);
        cudaMemset(D.scratch[s], 0, kScratchBytes);
      }
    }
    // peer access to every device initialised before this one (both ways)
    for (int o = 0; o < d; ++o) {
      if (devs_[o]->ordinal == D.ordinal) continue;  // two logical devices on one GPU: plain device copies
      int can = 0;
      cudaDeviceCanAccessPeer(&can, D.ordinal, devs_[o]->ordinal);
      if (can) {
        cudaDeviceEnablePeerAccess(devs_[o]->ordinal, 0);
        cudaSetDevice(devs_[o]->ordinal);
        cudaDeviceEnablePeerAccess(D.ordinal, 0);
        cudaSetDevice(D.ordinal);
      }
      cudaGetLastError();
    }
    // timestamp calibration: host CLOCK_MONOTONIC of the base event.  Logical
    // devices on the same GPU share the first one's base (one device clock), so
    // their timestamps compare exactly (violations() uses no slack for them)
    for (int o = 0; o < d; ++o)
      if (devs_[o]->ordinal == D.ordinal && devs_[o]->base) {
        D.base = devs_[o]->base;
        D.base_ns = devs_[o]->base_ns;
        D.base_shared = true;
        D.ready = true;
        return cuda_err(cudaGetLastError(), "device init", err);
      }
    e = cudaEventCreate(&D.base);
    if (e) return cuda_err(e, "cudaEventCreate", err);
    cudaEventRecord(D.base, D.streams[0]);
    cudaEventSynchronize(D.base);
    int64_t best = INT64_MAX;
    cudaEvent_t probe;
    cudaEventCreate(&probe);
    for (int k = 0; k < 5; ++k) {
      cudaEventRecord(probe, D.streams[0]);
      cudaEventSynchronize(probe);
      const int64_t host = now_ns();
      float ms = 0;
      cudaEventElapsedTime(&ms, D.base, probe);
      const int64_t b = host - static_cast<int64_t>(static_cast<double>(ms) * 1e6);
      if (b < best) best = b;
    }
    cudaEventDestroy(probe);
    D.base_ns = best;
    D.ready = true;
    return cuda_err(cudaGetLastError(), "device init", err);
  }

  void bind_thread(int d) override { cudaSetDevice(devs_[d]->ordinal); }
  bool same_clock(int a, int b) const override { return devs_[a]->ordinal == devs_[b]->ordinal; }
  uint64_t arena_capacity(int d) override { return devs_[d]->cap; }
  void* arena_ptr(int d, uint64_t off) override { return devs_[d]->arena + off; }

  void* event_create(int d, bool timing) override {
    Dev& D = *devs_[d];
    {
      std::lock_guard<std::mutex> g(D.pool_mu);
      auto& pool = timing ? D.pool_timing : D.pool_plain;
      if (!pool.empty()) {
        Ev* e = pool.back();
        pool.pop_back();
        return e;
      }
    }
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != D.ordinal) cudaSetDevice(D.ordinal);
    Ev* e = new Ev();
    e->timing = timing;
    cudaEventCreateWithFlags(&e->e, timing ? cudaEventDefault : cudaEventDisableTiming);
    if (cur != D.ordinal) cudaSetDevice(cur);
    return e;
  }
  void event_release(int d, void* ev) override {
    Dev& D = *devs_[d];
    std::lock_guard<std::mutex> g(D.pool_mu);
    Ev* e = static_cast<Ev*>(ev);
    if (shut_) {
      cudaEventDestroy(e->e);
      delete e;
      return;
    }
    (e->timing ? D.pool_timing : D.pool_plain).push_back(e);
  }
  int event_record(int d, int stream, void* ev, std::string& err) override {
    return cuda_err(cudaEventRecord(ev_of(ev), devs_[d]->streams[stream]), "cudaEventRecord", err);
  }
  int stream_wait(int d, int stream, void* ev, std::string& err) override {
    return cuda_err(cudaStreamWaitEvent(devs_[d]->streams[stream], ev_of(ev), 0),
                    "cudaStreamWaitEvent", err);
  }
  int event_sync(int, void* ev, std::string& err) override {
    return cuda_err(cudaEventSynchronize(ev_of(ev)), "kernel execution", err);
  }
  bool event_done(int, void* ev) override {
    const cudaError_t e = cudaEventQuery(ev_of(ev));
    if (e == cudaErrorNotReady) {
      cudaGetLastError();
      return false;
    }
    return true;
  }
  int event_query(int, void* ev, std::string& err) override {
    const cudaError_t e = cudaEventQuery(ev_of(ev));
    if (e == cudaSuccess) return 1;
    if (e == cudaErrorNotReady) {
      cudaGetLastError();
      return 0;
    }
    return cuda_err(e, "kernel execution", err);
  }
  int64_t event_time_ns(int d, void* ev) override {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, devs_[d]->base, ev_of(ev)) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return devs_[d]->base_ns + static_cast<int64_t>(static_cast<double>(ms) * 1e6);
  }
  int copy_h2d(int d, int stream, uint64_t dst, const void* src, uint64_t n, std::string& err) override {
    return cuda_err(cudaMemcpyAsync(devs_[d]->arena + dst, src, n, cudaMemcpyHostToDevice, devs_[d]->streams[stream]),
                    "H2D copy", err);
  }
  int copy_d2h(int d, int stream, void* dst, uint64_t src, uint64_t n, std::string& err) override {
    return cuda_err(cudaMemcpyAsync(dst, devs_[d]->arena + src, n, cudaMemcpyDeviceToHost, devs_[d]->streams[stream]),
                    "D2H copy", err);
  }
  int copy_p2p(int d, int stream, uint64_t dst, int sd, uint64_t src, uint64_t n, std::string& err) override {
    return cuda_err(cudaMemcpyPeerAsync(devs_[d]->arena + dst, devs_[d]->ordinal, devs_[sd]->arena + src,
                                        devs_[sd]->ordinal, n, devs_[d]->streams[stream]),
                    "peer copy", err);
  }
  uint64_t kernel_launches() const override { return g_kernel_launches.load(); }
  int status_alloc(int d) override {
    Dev& D = *devs_[d];
    std::lock_guard<std::mutex> g(D.pool_mu);
    if (D.status_free.empty()) return -1;
    const int k = D.status_free.back();
    D.status_free.pop_back();
    return k;
  }
  int status_take(int d, int slot) override {
    Dev& D = *devs_[d];
    std::lock_guard<std::mutex> g(D.pool_mu);
    volatile int* w = D.status + slot;
    const int v = *w;
    *w = 0;
    D.status_free.push_back(slot);
    return v;
  }
  bool supports(uint32_t op) const override {
    switch (op) {
      case SFX_OP_NOOP:
      case SFX_OP_SPIN:
      case SFX_OP_FAULT:
      case SFX_OP_CELL:
      case SFX_OP_BYTES_ADD:
      case SFX_OP_ADD_I64:
      case SFX_OP_EXTERN:
      case SFX_OP_DACC:
      case SFX_OP_FLUSH:
      case SFX_OP_ZERO:
      case SFX_OP_DGEMM:
      case SFX_OP_DSYRK:
      case SFX_OP_DTRSM:
      case SFX_OP_DPOTRF:
      case SFX_OP_P2P_PAIR:
      case SFX_OP_P2P_SELF:
      case SFX_OP_FILL_UNIFORM:
      case SFX_OP_FILL_SPD:
      case SFX_OP_FILL_PARTICLES:
        return true;
      default:
        return user_op(op) != nullptr;
    }
  }

  int launch(int d, int stream, const OpLaunch& op, std::string& err) override {
    set_deterministic_launches(op.deterministic);
    const int rc = launch_op(d, stream, op, err);
    set_deterministic_launches(false);
    return rc;
  }

  int launch_op(int d, int stream, const OpLaunch& op, std::string& err) {
    cudaStream_t s = devs_[d]->streams[stream];
    const Operand* o = op.o;
    auto f64 = [](const Operand& x) { return static_cast<double*>(x.dptr); };
    cudaError_t e = cudaSuccess;
    switch (op.op) {
      case SFX_OP_SPIN:
        e = launch_spin(op.ip[0], s);
        break;
      case SFX_OP_FAULT:
        e = launch_fault(static_cast<int>(op.ip[0]), s);
        break;
      case SFX_OP_ZERO:
        e = cudaMemsetAsync(o[0].dptr, 0, o[0].bytes, s);
        break;
      case SFX_OP_BYTES_ADD:
        e = launch_bytes_add(static_cast<unsigned char*>(o[0].dptr), op.ip[0], op.ip[1], op.ip[2], s);
        break;
      case SFX_OP_DACC: {
        const double* add[7];
        long long ld[7];
        for (int k = 1; k < op.n; ++k) {
          add[k - 1] = f64(o[k]);
          ld[k - 1] = o[k].ld;
        }
        e = launch_dacc(f64(o[0]), o[0].ld, o[0].rows, o[0].cols, add, ld, op.n - 1, s);
        break;
      }
      case SFX_OP_ADD_I64: {
        long long* cells[8];
        for (int k = 0; k < op.n; ++k) cells[k] = static_cast<long long*>(o[k].dptr);
        e = launch_add_i64(cells, op.n, op.ip[0], s);
        break;
      }
      case SFX_OP_CELL: {
        const long long* reads[7];
        for (int k = 1; k < op.n; ++k) reads[k - 1] = static_cast<const long long*>(o[k].dptr);
        e = launch_cell(static_cast<long long*>(o[0].dptr), reads, op.n - 1, op.ip[0], op.ip[1], op.ip[2], s);
        break;
      }
      case SFX_OP_FILL_UNIFORM:
        e = launch_fill_uniform(f64(o[0]), o[0].rows, o[0].cols, o[0].ld, op.ip[0], op.ip[1], op.ip[2], op.ip[3], s);
        break;
      case SFX_OP_FILL_SPD:
        e = launch_fill_spd(f64(o[0]), o[0].rows, o[0].cols, o[0].ld, op.ip[0], op.ip[1], op.ip[2], op.ip[3], s);
        break;
      case SFX_OP_FILL_PARTICLES:
        e = launch_fill_particles(f64(o[0]), o[0].cols, o[0].ld, op.ip[0], op.ip[1], s);
        break;
      case SFX_OP_DGEMM: {
        const bool tb = op.ip[0] != 0;
        e = launch_dgemm(f64(o[0]), o[0].ld, f64(o[1]), o[1].ld, f64(o[2]), o[2].ld, static_cast<int>(o[2].rows),
                         static_cast<int>(o[2].cols), static_cast<int>(o[0].cols), op.fp[0], op.fp[1], tb, false, s);
        break;
      }
      case SFX_OP_DSYRK:
        e = launch_dgemm(f64(o[0]), o[0].ld, f64(o[0]), o[0].ld, f64(o[1]), o[1].ld, static_cast<int>(o[1].rows),
                         static_cast<int>(o[1].rows), static_cast<int>(o[0].cols), op.fp[0], op.fp[1], true, true, s);
        break;
      case SFX_OP_DTRSM:
        if (op.ip[0] == 2) {
          const size_t need = static_cast<size_t>(o[1].rows) * o[1].cols * 8;
          void* sc = trsm_scratch(d, stream, need);
          if (!sc) {
            err = "trsm scratch allocation failed";
            return SFX_ERR_CUDA;
          }
          e = launch_dtrsm_fullinv(f64(o[0]), o[0].ld, f64(o[1]), o[1].ld, static_cast<int>(o[1].rows),
                                   static_cast<int>(o[1].cols), sc, need, s);
        } else if (op.ip[0] && coop_supported(static_cast<int>(o[1].rows), static_cast<int>(o[1].cols))) {
          TrsmDesc td{f64(o[0]), o[0].ld, f64(o[1]), o[1].ld};
          e = launch_dtrsm_inv_group(&td, 1, static_cast<int>(o[1].rows), static_cast<int>(o[1].cols), s);
        } else if (devs_[d]->scratch[stream] &&
                   coop_supported(static_cast<int>(o[1].rows), static_cast<int>(o[1].cols))) {
          TrsmDesc td{f64(o[0]), o[0].ld, f64(o[1]), o[1].ld};
          e = launch_dtrsm_coop_group(&td, 1, static_cast<int>(o[1].rows), static_cast<int>(o[1].cols),
                                      devs_[d]->scratch[stream], kScratchBytes, s);
        } else {
          e = launch_dtrsm(f64(o[0]), o[0].ld, f64(o[1]), o[1].ld, static_cast<int>(o[1].rows),
                           static_cast<int>(o[1].cols), s);
        }
        break;
      case SFX_OP_DPOTRF: {
        int* info = status_ptr(d, op.status_slot);
        static const bool old_potrf = getenv("SFX_POTRF") && !strcmp(getenv("SFX_POTRF"), "coop");  // A/B only
        if (!old_potrf && devs_[d]->scratch[stream] && flow_supported(static_cast<int>(o[0].rows)) &&
            o[0].ld % 2 == 0)
          e = launch_dpotrf_flow(f64(o[0]), o[0].ld, static_cast<int>(o[0].rows), info, devs_[d]->scratch[stream],
                                 kScratchBytes, s, op.ip[0]);
        else if (op.ip[0] == 2 && devs_[d]->scratch[stream] && fullinv_supported(static_cast<int>(o[0].rows)))
          e = launch_dpotrf_fullinv(f64(o[0]), o[0].ld, static_cast<int>(o[0].rows), info, devs_[d]->scratch[stream],
                                    kScratchBytes, s);
        else if (devs_[d]->scratch[stream] && coop_supported(static_cast<int>(o[0].rows), static_cast<int>(o[0].rows)))
          e = launch_dpotrf_coop(f64(o[0]), o[0].ld, static_cast<int>(o[0].rows), info, devs_[d]->scratch[stream], s,
                                 op.ip[0] != 0);
        else
          e = launch_dpotrf(f64(o[0]), o[0].ld, static_cast<int>(o[0].rows), info, s);
        break;
      }
      case SFX_OP_P2P_PAIR:
        e = launch_p2p(f64(o[0]), o[0].ld, static_cast<int>(o[0].cols), f64(o[1]), o[1].ld, static_cast<int>(o[1].cols),
                       f64(o[2]), o[2].ld, f64(o[3]), o[3].ld, false, op.fp[0], s);
        break;
      case SFX_OP_P2P_SELF:
        e = launch_p2p(f64(o[0]), o[0].ld, static_cast<int>(o[0].cols), nullptr, 0, 0, f64(o[1]), o[1].ld, nullptr, 0,
                       true, op.fp[0], s);
        break;
      default: {
        const UserOp* u = user_op(op.op);
        if (!u) {
          err = "unsupported op";
          return SFX_ERR_UNSUPPORTED;
        }
        cudaGetLastError();  // a launch error left by the launcher is its own
        const int rc = run_user_op(*u, op, d, s, err);
        if (rc) return rc;
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_err(e, (std::string("user op '") + u->name + "' launch").c_str(), err);
        break;
      }
    }
    return cuda_err(e, "kernel launch", err);
  }

  int launch_group(int d, int stream, const std::vector<OpLaunch>& ops, std::string& err) override {
    set_deterministic_launches(ops[0].deterministic);
    const int rc = launch_group_op(d, stream, ops, err);
    set_deterministic_launches(false);
    return rc;
  }

  int launch_group_op(int d, int stream, const std::vector<OpLaunch>& ops, std::string& err) {
    const OpLaunch& f = ops[0];
    if (ops.size() > 1 && (f.op == SFX_OP_DGEMM || f.op == SFX_OP_DSYRK)) {
      std::vector<GemmDesc> g(ops.size());
      const bool syrk = f.op == SFX_OP_DSYRK;
      for (size_t i = 0; i < ops.size(); ++i) {
        const Operand* o = ops[i].o;
        if (syrk)
          g[i] = GemmDesc{static_cast<const double*>(o[0].dptr), o[0].ld, static_cast<const double*>(o[0].dptr),
                          o[0].ld, static_cast<double*>(o[1].dptr), o[1].ld};
        else
          g[i] = GemmDesc{static_cast<const double*>(o[0].dptr), o[0].ld, static_cast<const double*>(o[1].dptr),
                          o[1].ld, static_cast<double*>(o[2].dptr), o[2].ld};
      }
      const Operand* o = f.o;
      cudaError_t e =
          syrk ? launch_dgemm_group(g.data(), static_cast<int>(g.size()), static_cast<int>(o[1].rows),
                                    static_cast<int>(o[1].rows), static_cast<int>(o[0].cols), f.fp[0], f.fp[1], true,
                                    true, devs_[d]->streams[stream])
               : launch_dgemm_group(g.data(), static_cast<int>(g.size()), static_cast<int>(o[2].rows),
                                    static_cast<int>(o[2].cols), static_cast<int>(o[0].cols), f.fp[0], f.fp[1],
                                    f.ip[0] != 0, false, devs_[d]->streams[stream]);
      return cuda_err(e, "grouped dgemm launch", err);
    }
    if (ops.size() > 1 && (f.op == SFX_OP_P2P_PAIR || f.op == SFX_OP_P2P_SELF)) {
      const bool self = f.op == SFX_OP_P2P_SELF;
      std::vector<P2PDesc> pd(ops.size());
      for (size_t i = 0; i < ops.size(); ++i) {
        const Operand* o = ops[i].o;
        auto f64p = [](const Operand& x) { return static_cast<double*>(x.dptr); };
        if (self)
          pd[i] = P2PDesc{f64p(o[0]), o[0].ld, static_cast<int>(o[0].cols), nullptr, 0, 0, f64p(o[1]), o[1].ld,
                          nullptr, 0};
        else
          pd[i] = P2PDesc{f64p(o[0]), o[0].ld, static_cast<int>(o[0].cols), f64p(o[1]), o[1].ld,
                          static_cast<int>(o[1].cols), f64p(o[2]), o[2].ld, f64p(o[3]), o[3].ld};
      }
      cudaError_t e = launch_p2p_group(pd.data(), static_cast<int>(pd.size()), self, f.fp[0], devs_[d]->streams[stream]);
      return cuda_err(e, "grouped p2p launch", err);
    }
    if (ops.size() > 1 && f.op == SFX_OP_SPIN) {  // members share ip[0] (same_signature)
      cudaError_t e = launch_spin_group(static_cast<int>(ops.size()), f.ip[0], devs_[d]->streams[stream]);
      return cuda_err(e, "grouped spin launch", err);
    }
    if (ops.size() > 1 && f.op == SFX_OP_DTRSM && f.ip[0] == 2) {
      // grouped full-inverse TRSMs: X_i = B_i W_i^T for every member in ONE TRI-masked
      // DGEMM launch (beta = 0, no split-K: no scratch memset, no atomics), then
      // each X_i copied back over B_i
      const size_t one = static_cast<size_t>(f.o[1].rows) * f.o[1].cols * 8;
      double* X = static_cast<double*>(trsm_scratch(d, stream, one * ops.size()));
      if (!X) {
        // not enough memory beside the arena for the group's scratch: one TRSM at
        // a time (each needs a single tile of scratch)
        for (const OpLaunch& op : ops) {
          const int rc = launch(d, stream, op, err);
          if (rc) return rc;
        }
        return SFX_OK;
      }
      const long long ldx = f.o[1].cols;
      std::vector<GemmDesc> g(ops.size());
      for (size_t i = 0; i < ops.size(); ++i)
        g[i] = GemmDesc{static_cast<const double*>(ops[i].o[1].dptr), ops[i].o[1].ld,
                        static_cast<const double*>(ops[i].o[0].dptr), ops[i].o[0].ld, X + i * (one / 8), ldx};
      const int M = static_cast<int>(f.o[1].rows), n = static_cast<int>(f.o[1].cols);
      cudaError_t e = launch_dgemm_group(g.data(), static_cast<int>(g.size()), M, n, n, 1.0, 0.0, false, false,
                                         devs_[d]->streams[stream], true);
      for (size_t i = 0; i < ops.size() && e == cudaSuccess; ++i)
        e = cudaMemcpy2DAsync(ops[i].o[1].dptr, ops[i].o[1].ld * 8, X + i * (one / 8), ldx * 8, ldx * 8, M,
                              cudaMemcpyDeviceToDevice, devs_[d]->streams[stream]);
      return cuda_err(e, "grouped full-inverse dtrsm launch", err);
    }
    if (ops.size() > 1 && f.op == SFX_OP_DTRSM && f.ip[0]) {
      std::vector<TrsmDesc> td(ops.size());
      for (size_t i = 0; i < ops.size(); ++i)
        td[i] = TrsmDesc{static_cast<const double*>(ops[i].o[0].dptr), ops[i].o[0].ld,
                         static_cast<double*>(ops[i].o[1].dptr), ops[i].o[1].ld};
      cudaError_t e = launch_dtrsm_inv_group(td.data(), static_cast<int>(td.size()), static_cast<int>(f.o[1].rows),
                                             static_cast<int>(f.o[1].cols), devs_[d]->streams[stream]);
      return cuda_err(e, "grouped dtrsm (inverse blocks) launch", err);
    }
    if (ops.size() > 1 && f.op == SFX_OP_DTRSM && devs_[d]->scratch[stream]) {
      std::vector<TrsmDesc> td(ops.size());
      for (size_t i = 0; i < ops.size(); ++i)
        td[i] = TrsmDesc{static_cast<const double*>(ops[i].o[0].dptr), ops[i].o[0].ld,
                         static_cast<double*>(ops[i].o[1].dptr), ops[i].o[1].ld};
      cudaError_t e = launch_dtrsm_coop_group(td.data(), static_cast<int>(td.size()), static_cast<int>(f.o[1].rows),
                                              static_cast<int>(f.o[1].cols), devs_[d]->scratch[stream],
                                              kScratchBytes, devs_[d]->streams[stream]);
      return cuda_err(e, "grouped cooperative dtrsm launch", err);
    }
    for (const OpLaunch& op : ops) {
      int rc = launch(d, stream, op, err);
      if (rc) return rc;
    }
    return SFX_OK;
  }

  void shutdown() override {
    if (shut_) return;
    for (Dev* dp : devs_) {
      Dev& D = *dp;
      if (!D.ready) continue;
      cudaSetDevice(D.ordinal);
      cudaDeviceSynchronize();
      std::lock_guard<std::mutex> g(D.pool_mu);
      for (Ev* e : D.pool_timing) {
        cudaEventDestroy(e->e);
        delete e;
      }
      for (Ev* e : D.pool_plain) {
        cudaEventDestroy(e->e);
        delete e;
      }
      D.pool_timing.clear();
      D.pool_plain.clear();
      if (D.base && !D.base_shared) cudaEventDestroy(D.base);
      for (auto st : D.streams) cudaStreamDestroy(st);
      D.streams.clear();
      if (D.arena) cudaFree(D.arena);
      if (D.status) cudaFreeHost(D.status);
      D.status = nullptr;
      for (void* p : D.scratch)
        if (p) cudaFree(p);
      D.scratch.clear();
      for (void* p : D.tscratch)
        if (p) cudaFree(p);
      D.tscratch.clear();
      D.arena = nullptr;
      D.ready = false;
    }
    shut_ = true;
  }

 private:
  std::vector<Dev*> devs_;
  bool shut_ = false;
};

}  // namespace

Backend* make_cuda_backend(int ndev, const int* ordinals, bool) { return new CudaBackend(ndev, ordinals); }

}  // namespace sfx
