// Host-memory simulated devices.
//
// Mirrors the reference's own simulated accelerator (a bytearray arena per
// device, reference src/device.py:78-116) so the native runtime's
// dependency core, LRU arena and coherency logic can be exercised through the
// C ABI on a machine without a GPU.  It executes only the runtime's
// bookkeeping test ops (noop, spin, the int64 cell arithmetic of the
// reference's random programs, byte adds, zero).  Every tile op (DGEMM, DSYRK,
// DTRSM, DPOTRF, particles, generators) is refused at submit time with
// SFX_ERR_UNSUPPORTED: there is no CPU fallback for the hot path.
#include <cstdlib>
#include <cstring>

#include "runtime.h"

namespace sfx {
namespace {

constexpr int64_t kMod = 10000019;  // reference tests/conftest.py:22

inline int64_t pymod(int64_t x) { return ((x % kMod) + kMod) % kMod; }

struct SimEvent {
  int64_t t = 0;
};

class SimBackend : public Backend {
 public:
  explicit SimBackend(int ndev) : arenas_(ndev, nullptr), caps_(ndev, 0) {}
  ~SimBackend() override { shutdown(); }
  bool is_sim() const override { return true; }
  int init_device(int d, int, int, int, int, int, uint64_t bytes, std::string& err) override {
    if (!bytes) bytes = 16ull << 20;  // reference default device_memory (engine.py:180)
    const uint64_t alloc = (bytes + 63) / 64 * 64;
    arenas_[d] = static_cast<uint8_t*>(aligned_alloc(64, alloc));
    if (!arenas_[d]) {
      err = "sim arena allocation failed";
      return SFX_ERR_STAGING;
    }
    memset(arenas_[d], 0, alloc);
    caps_[d] = bytes;
    return SFX_OK;
  }
  void bind_thread(int) override {}
  uint64_t arena_capacity(int d) override { return caps_[d]; }
  void* arena_ptr(int d, uint64_t off) override { return arenas_[d] + off; }
  void* event_create(int, bool) override { return new SimEvent(); }
  void event_release(int, void* ev) override { delete static_cast<SimEvent*>(ev); }
  int event_record(int, int, void* ev, std::string&) override {
    static_cast<SimEvent*>(ev)->t = now_ns();
    return SFX_OK;
  }
  int stream_wait(int, int, void*, std::string&) override { return SFX_OK; }
  int event_sync(int, void*, std::string&) override { return SFX_OK; }
  bool event_done(int, void*) override { return true; }
  int64_t event_time_ns(int, void* ev) override { return static_cast<SimEvent*>(ev)->t; }
  int copy_h2d(int d, int, uint64_t dst, const void* src, uint64_t n, std::string&) override {
    memcpy(arenas_[d] + dst, src, n);
    return SFX_OK;
  }
  int copy_d2h(int d, int, void* dst, uint64_t src, uint64_t n, std::string&) override {
    memcpy(dst, arenas_[d] + src, n);
    return SFX_OK;
  }
  int copy_p2p(int d, int, uint64_t dst, int sd, uint64_t src, uint64_t n, std::string&) override {
    memcpy(arenas_[d] + dst, arenas_[sd] + src, n);
    return SFX_OK;
  }
  bool supports(uint32_t op) const override {
    switch (op) {
      case SFX_OP_NOOP:
      case SFX_OP_SPIN:
      case SFX_OP_CELL:
      case SFX_OP_BYTES_ADD:
      case SFX_OP_ADD_I64:
      case SFX_OP_EXTERN:
      case SFX_OP_FLUSH:
      case SFX_OP_ZERO:
        return true;
      default:
        return user_op(op) != nullptr;
    }
  }
  int launch(int d, int, const OpLaunch& op, std::string& err) override {
    switch (op.op) {
      case SFX_OP_NOOP:
        return SFX_OK;
      case SFX_OP_SPIN: {
        const int64_t until = now_ns() + op.ip[0];
        while (now_ns() < until) {
        }
        return SFX_OK;
      }
      case SFX_OP_ZERO:
        memset(op.o[0].dptr, 0, op.o[0].bytes);
        return SFX_OK;
      case SFX_OP_ADD_I64:
        for (int k = 0; k < op.n; ++k)
          __atomic_fetch_add(static_cast<int64_t*>(op.o[k].dptr), op.ip[0], __ATOMIC_RELAXED);
        return SFX_OK;
      case SFX_OP_BYTES_ADD: {
        uint8_t* p = static_cast<uint8_t*>(op.o[0].dptr);
        for (int64_t i = op.ip[0]; i < op.ip[0] + op.ip[1]; ++i)
          p[i] = static_cast<uint8_t>((static_cast<int64_t>(p[i]) + op.ip[2]) & 255);
        return SFX_OK;
      }
      case SFX_OP_CELL: {
        int64_t* t = static_cast<int64_t*>(op.o[0].dptr);
        int64_t rsum = 0;
        for (int k = 1; k < op.n; ++k) rsum += *static_cast<int64_t*>(op.o[k].dptr);
        const int64_t kind = op.ip[0], a = op.ip[1], b = op.ip[2];
        switch (kind) {
          case 0:
            break;
          case 1:
            *t = pymod(a * *t + b + rsum);
            break;
          case 2:
            if (*t % 2 == 0) *t = pymod(a * *t + b + rsum);
            break;
          case 3:
            *t = pymod(*t + pymod(b + rsum));
            break;
          case 4:
            *t = pymod(*t + b + a * rsum);
            break;
          default:
            err = "bad cell op kind";
            return SFX_ERR_CONFIG;
        }
        return SFX_OK;
      }
      default:
        if (const UserOp* u = user_op(op.op)) return run_user_op(*u, op, d, nullptr, err);  // host pointers
        err = "op not available on the simulated backend";
        return SFX_ERR_UNSUPPORTED;
    }
  }
  void shutdown() override {
    for (auto& a : arenas_) {
      free(a);
      a = nullptr;
    }
  }

 private:
  std::vector<uint8_t*> arenas_;
  std::vector<uint64_t> caps_;
};

}  // namespace

Backend* make_sim_backend(int ndev) { return new SimBackend(ndev); }

}  // namespace sfx
