// Native STF runtime (see runtime.h for the reference mapping).
#include "runtime.h"

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <ctime>

namespace sfx {

int64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return static_cast<int64_t>(ts.tv_sec) * 1000000000LL + ts.tv_nsec;
}

Sync::~Sync() {
  if (be && event) be->event_release(dev, event);
}

static bool heap_less(const Task* a, const Task* b) {
  // max-heap on (priority, -seq): higher priority first, FIFO among equals
  if (a->prio != b->prio) return a->prio < b->prio;
  return a->seq > b->seq;
}

void DevQueue::push(Task* t) {
  if (!prio) {
    fifo.push_back(t);
  } else {
    heap.push_back(t);
    std::push_heap(heap.begin(), heap.end(), heap_less);
  }
}

void DevQueue::push_front(Task* t) {
  if (!prio)
    fifo.push_front(t);
  else
    push(t);  // heap order is (priority, seq): re-pushing restores its place
}

Task* DevQueue::peek() const {
  if (!prio) return fifo.empty() ? nullptr : fifo.front();
  return heap.empty() ? nullptr : heap.front();
}

Task* DevQueue::pop() {
  if (!prio) {
    if (fifo.empty()) return nullptr;
    Task* t = fifo.front();
    fifo.pop_front();
    return t;
  }
  if (heap.empty()) return nullptr;
  std::pop_heap(heap.begin(), heap.end(), heap_less);
  Task* t = heap.back();
  heap.pop_back();
  return t;
}

static std::string fmt(const char* f, ...) __attribute__((format(printf, 1, 2)));
static std::string fmt(const char* f, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof buf, f, ap);
  va_end(ap);
  return buf;
}

// ---- user ops (sfx_register_op) ---------------------------------------------
static UserOp g_user_ops[SFX_OP_USER_MAX];
static std::atomic<uint32_t> g_user_count{0};
static std::mutex g_user_mu;

const UserOp* user_op(uint32_t op) {
  if (op < SFX_OP_USER_BASE) return nullptr;
  const uint32_t k = op - SFX_OP_USER_BASE;
  return k < g_user_count.load(std::memory_order_acquire) ? &g_user_ops[k] : nullptr;
}

int register_user_op(const char* name, sfx_user_launch_fn fn, void* user, uint32_t* op, std::string& err) {
  if (!name || !*name || strlen(name) >= sizeof(UserOp::name) || !fn) {
    err = "sfx_register_op: needs a name of 1..63 characters and a launcher";
    return SFX_ERR_CONFIG;
  }
  std::lock_guard<std::mutex> g(g_user_mu);
  const uint32_t n = g_user_count.load(std::memory_order_relaxed);
  for (uint32_t k = 0; k < n; ++k)
    if (!strcmp(g_user_ops[k].name, name)) {
      err = fmt("sfx_register_op: an op named '%s' is already registered", name);
      return SFX_ERR_CONFIG;
    }
  if (n >= SFX_OP_USER_MAX) {
    err = fmt("sfx_register_op: at most %d user ops", SFX_OP_USER_MAX);
    return SFX_ERR_CONFIG;
  }
  UserOp& u = g_user_ops[n];
  snprintf(u.name, sizeof u.name, "%s", name);
  u.fn = fn;
  u.user = user;
  g_user_count.store(n + 1, std::memory_order_release);  // publishes the entry
  *op = SFX_OP_USER_BASE + n;
  return SFX_OK;
}

int run_user_op(const UserOp& u, const OpLaunch& op, int dev, void* stream, std::string& err) {
  sfx_view v[8];
  for (int k = 0; k < op.n; ++k) {
    const Operand& o = op.o[k];
    v[k] = sfx_view{o.dptr, o.bytes, o.rows, o.cols, o.ld, o.dtype, o.mode, dev, 0};
  }
  const int rc = u.fn(v, op.n, stream, op.fp, op.ip, u.user);
  if (rc) {
    err = fmt("user op '%s' failed (launcher returned %d)", u.name, rc);
    return SFX_ERR_USER;
  }
  return SFX_OK;
}

Runtime::Runtime(Backend* be, int ndev, int nstreams, uint32_t sched, uint32_t flags, uint32_t window,
                 uint64_t align)
    : be_(be),
      ndev_(ndev),
      nstreams_(nstreams),
      sched_(sched),
      flags_(flags),
      window_(window ? window : 4096u),
      align_(align),
      trace_((flags & SFX_FLAG_TRACE) != 0),
      ktime_((flags & (SFX_FLAG_TRACE | SFX_FLAG_KTIME)) != 0) {
  paused_ = (flags & SFX_FLAG_PAUSED) != 0;
  nurgent_ = nstreams >= 2 ? std::max(2, nstreams / 4) : 0;
  const char* rm = getenv("SFX_SUBMIT_RING");
  ring_mode_ = !(rm && rm[0] == '0');
}

int Runtime::init(const uint64_t* arena_bytes, std::string& err) {
  for (int d = 0; d < ndev_; ++d) {
    auto dev = std::make_unique<Device>();
    dev->index = d;
    dev->queue.prio = sched_ == SFX_SCHED_PRIO;
    if (be_->is_sim()) {
      ncoop_ = 0;
      prefetch_ = false;  // keeps the simulator's LRU behaviour identical to the reference
    }
    dev->stream_inflight.assign(nstreams_ + nurgent_ + ncoop_ + 1, 0);
    dev->stream_groups.assign(nstreams_ + nurgent_ + ncoop_ + 1, 0);
    int rc = be_->init_device(d, d, nstreams_, nurgent_, ncoop_, 1, arena_bytes ? arena_bytes[d] : 0, err);
    if (rc) return rc;
    dev->capacity = be_->arena_capacity(d);
    dev->free_bytes = dev->capacity;
    dev->free_list[0] = dev->capacity;
    dev->stats.capacity = dev->capacity;
    devs_.push_back(std::move(dev));
  }
  for (int d = 0; d < ndev_; ++d) {
    devs_[d]->exec_thread = std::thread(&Runtime::exec_loop, this, d);
    if (!be_->is_sim()) devs_[d]->comp_thread = std::thread(&Runtime::comp_loop, this, d);
  }
  started_ = true;
  return SFX_OK;
}

Runtime::~Runtime() {
  {
    std::unique_lock<std::mutex> lk(mu_);
    stopping_ = true;
    for (auto& d : devs_) {
      d->exec_cv.notify_all();
      d->comp_cv.notify_all();
    }
    done_cv_.notify_all();
    extern_cv_.notify_all();
  }
  for (auto& d : devs_) {
    if (d->exec_thread.joinable()) d->exec_thread.join();
    if (d->comp_thread.joinable()) d->comp_thread.join();
  }
  // drop every sync/event reference before the backend goes away
  for (auto& t : task_store_) {
    t->waits.clear();
    t->start.reset();
    t->end.reset();
    t->copy_syncs.clear();
  }
  for (auto& h : handle_store_) {
    h->host_ready.reset();
    h->commute_last.reset();
    for (Block* b : h->blocks) {
      if (b) {
        b->ready.reset();
        delete b;
      }
    }
    h->blocks.clear();
  }
  for (auto& d : devs_) d->pending_wb.clear();
  be_->shutdown();
  delete be_;
}

// ---------------------------------------------------------------- graphs

int Runtime::graph_create(uint32_t* gid) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  auto g = std::make_unique<Graph>();
  g->gid = next_gid_++;
  *gid = g->gid;
  graphs_[g->gid] = std::move(g);
  return SFX_OK;
}

int Runtime::reg(uint32_t gid, uint64_t hid, void* host, uint64_t bytes, int64_t rows, int64_t cols, int64_t ld,
                 int32_t dtype) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  auto git = graphs_.find(gid);
  if (git == graphs_.end()) {
    last_error = fmt("unknown graph %u", gid);
    return SFX_ERR_CONFIG;
  }
  if (handles_.count(hid)) {
    last_error = fmt("handle %llu is already registered", (unsigned long long)hid);
    return SFX_ERR_REGISTRATION;
  }
  // One host buffer, one live handle across graphs.  The reference registry is
  // per graph (graph.py:35) and its device arenas key blocks by hid, so the same
  // object in two graphs has two device copies; with device caches that outlive
  // a graph's work, an old graph's dirty copy written back later would clobber
  // what the new graph staged.  The older handle is retired here: its dirty copy
  // is written home and its blocks dropped, and the old graph can no longer use
  // it.  If it still has pending accesses the registration fails instead (wait
  // for the old graph first).  Handles of the SAME graph may overlap (array
  // views and their whole object, reference access.py:103-129).
  if (host && bytes) {
    const uintptr_t lo = reinterpret_cast<uintptr_t>(host), hi = lo + bytes;
    std::vector<Handle*> olds;
    for (auto it = host_ranges_.lower_bound(hi); it != host_ranges_.begin();) {
      --it;
      if (it->first + max_handle_bytes_ <= lo) break;
      Handle* o = it->second;
      if (it->first + o->bytes > lo && o->gid != gid) olds.push_back(o);
    }
    for (Handle* o : olds) {
      bool busy = o->active < o->slot_end();
      for (Block* b : o->blocks) busy = busy || (b && b->pins > 0);
      if (busy) {
        last_error = fmt("the object's memory is still in use by graph %u (pending accesses): wait for that graph "
                         "before registering the object in another graph", o->gid);
        return SFX_ERR_REGISTRATION;
      }
    }
    for (Handle* o : olds) {
      int rc = retire_blocks(o);
      if (rc) return rc;
      o->superseded = true;
      for (auto it = host_ranges_.begin(); it != host_ranges_.end(); ++it)
        if (it->second == o) {
          host_ranges_.erase(it);
          break;
        }
    }
  }
  auto h = std::make_unique<Handle>();
  h->hid = hid;
  h->gid = gid;
  h->host = host;
  h->bytes = bytes;
  h->rows = rows;
  h->cols = cols;
  h->ld = ld;
  h->dtype = dtype;
  h->blocks.assign(ndev_, nullptr);
  h->graph = git->second.get();
  handles_[hid] = h.get();
  if (host && bytes) {
    host_ranges_.emplace(reinterpret_cast<uintptr_t>(host), h.get());
    max_handle_bytes_ = std::max(max_handle_bytes_, bytes);
  }
  git->second->handles.push_back(h.get());
  handle_store_.push_back(std::move(h));
  return SFX_OK;
}

int Runtime::set_home(uint64_t hid, int dev) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  auto it = handles_.find(hid);
  if (it == handles_.end()) {
    last_error = "set_home: unknown handle";
    return SFX_ERR_REGISTRATION;
  }
  it->second->home = (dev >= 0 && ndev_ > 0) ? dev % ndev_ : -1;
  return SFX_OK;
}

int Runtime::retire_blocks(Handle* h) {
  // caller holds mu_ and checked that no block is pinned
  for (int d = 0; d < ndev_; ++d) {
    Block* b = h->blocks[d];
    if (!b) continue;
    if (b->dirty) {
      // synchronous write-back: the host object is the only copy left afterwards
      std::string err;
      be_->bind_thread(d);
      if (b->ready && !b->ready->complete) be_->event_sync(d, b->ready->event, err);
      void* ev = be_->event_create(d, false);
      int rc = be_->copy_d2h(d, 0, h->host, b->off, h->bytes, err);
      if (!rc) rc = be_->event_record(d, 0, ev, err);
      if (!rc) rc = be_->event_sync(d, ev, err);
      be_->event_release(d, ev);
      if (rc) {
        last_error = err;
        return SFX_ERR_CUDA;
      }
      devs_[d]->stats.bytes_from_device += h->bytes;
      devs_[d]->stats.copies_from_device += 1;
      h->host_valid = true;
      h->dirty_dev = -1;
    }
    drop_block(b, false, nullptr, 0);
  }
  return SFX_OK;
}

int Runtime::unreg(uint64_t hid) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  auto it = handles_.find(hid);
  if (it == handles_.end()) {
    last_error = "object is not registered";
    return SFX_ERR_REGISTRATION;
  }
  Handle* h = it->second;
  if (h->active < h->slot_end()) {
    // handles.py:179-182
    last_error = "cannot unregister an object with pending accesses";
    return SFX_ERR_REGISTRATION;
  }
  for (Block* b : h->blocks)
    if (b && b->pins > 0) {
      last_error = "cannot unregister an object still in use on a device";
      return SFX_ERR_REGISTRATION;
    }
  int rc = retire_blocks(h);
  if (rc) return rc;
  for (auto r = host_ranges_.begin(); r != host_ranges_.end(); ++r)
    if (r->second == h) {
      host_ranges_.erase(r);
      break;
    }
  handles_.erase(it);
  return SFX_OK;
}

// ------------------------------------------------------------- insertion

// DPOTRF / DTRSM with the full triangular inverse (factor_inv.cu): exact doubling
// over 64-blocks, and small enough for the cooperative factorization
static bool fullinv_size(int64_t n) {
  if (n < 128 || n > 2048 || n % 64) return false;
  const int64_t nb = n / 64;
  return (nb & (nb - 1)) == 0;
}

static int expect_f64(const Handle* h, const char* what, std::string& err) {
  if (h->dtype != SFX_DTYPE_F64 || h->rows <= 0 || h->cols <= 0 || h->ld < h->cols ||
      h->bytes < static_cast<uint64_t>((h->rows - 1) * h->ld + h->cols) * 8) {
    err = fmt("%s must be a 2-D float64 tile (got dtype %d, %lldx%lld ld %lld)", what, h->dtype,
              (long long)h->rows, (long long)h->cols, (long long)h->ld);
    return SFX_ERR_CONFIG;
  }
  return 0;
}

int Runtime::validate(const sfx_task_desc& d, const sfx_access* acc, std::string& err) {
  if (!graphs_.count(d.graph)) {
    err = fmt("unknown graph %u", d.graph);
    return SFX_ERR_CONFIG;
  }
  if (!be_->supports(d.op)) {
    err = fmt("op %u needs a CUDA device: the simulated backend only runs the runtime's test ops", d.op);
    return SFX_ERR_UNSUPPORTED;
  }
  std::vector<Handle*> hs(d.n_access);
  for (uint32_t k = 0; k < d.n_access; ++k) {
    auto it = handles_.find(acc[k].hid);
    if (it == handles_.end()) {
      err = fmt("access %u names unregistered handle %llu", k, (unsigned long long)acc[k].hid);
      return SFX_ERR_REGISTRATION;
    }
    if (acc[k].mode > SFX_MAYBE_WRITE) {
      err = fmt("bad access mode %u", acc[k].mode);
      return SFX_ERR_CONFIG;
    }
    hs[k] = it->second;
    if (hs[k]->superseded) {
      err = fmt("handle %llu: its object was registered by another graph since (one live registration per host "
                "buffer); register it again in this graph", (unsigned long long)acc[k].hid);
      return SFX_ERR_REGISTRATION;
    }
    for (uint32_t j = 0; j < k; ++j)
      if (hs[j] == hs[k]) {
        err = "task declares the same object twice";  // graph.py:134-137
        return SFX_ERR_DUPLICATE;
      }
  }
  auto need = [&](uint32_t n) {
    if (d.n_access != n) {
      err = fmt("op %u takes %u accesses, got %u", d.op, n, d.n_access);
      return false;
    }
    return true;
  };
  auto writes = [&](uint32_t k) {
    if (!mode_writes(acc[k].mode)) {
      err = fmt("op %u writes operand %u but it is declared read-only", d.op, k);
      return false;
    }
    return true;
  };
  int rc;
  switch (d.op) {
    case SFX_OP_NOOP:
    case SFX_OP_SPIN:
    case SFX_OP_FAULT:
      return 0;
    case SFX_OP_CELL:
      if (d.n_access < 1 || d.n_access > 8) {
        err = "cell op takes a target plus up to 7 read cells";
        return SFX_ERR_CONFIG;
      }
      for (uint32_t k = 0; k < d.n_access; ++k)
        if (hs[k]->bytes < 8) {
          err = "cell op operands must be 8-byte int64 cells";
          return SFX_ERR_CONFIG;
        }
      return 0;
    case SFX_OP_ADD_I64:
      if (d.n_access < 1 || d.n_access > 8) {
        err = "add_i64 takes 1 to 8 int64 cells";
        return SFX_ERR_CONFIG;
      }
      for (uint32_t k = 0; k < d.n_access; ++k)
        if (hs[k]->bytes < 8 || !mode_writes(acc[k].mode)) {
          err = "add_i64 operands must be written 8-byte int64 cells";
          return SFX_ERR_CONFIG;
        }
      return 0;
    case SFX_OP_BYTES_ADD:
      if (!need(1) || !writes(0)) return SFX_ERR_CONFIG;
      if (d.iparam[0] < 0 || d.iparam[1] < 0 || static_cast<uint64_t>(d.iparam[0] + d.iparam[1]) > hs[0]->bytes) {
        err = "bytes_add range outside the buffer";
        return SFX_ERR_CONFIG;
      }
      return 0;
    case SFX_OP_ZERO:
      if (!need(1) || !writes(0)) return SFX_ERR_CONFIG;
      return 0;
    case SFX_OP_FILL_UNIFORM:
    case SFX_OP_FILL_SPD:
    case SFX_OP_FILL_PARTICLES:
      if (!need(1) || !writes(0)) return SFX_ERR_CONFIG;
      return expect_f64(hs[0], "fill target", err);
    case SFX_OP_DGEMM: {
      if (!need(3) || !writes(2)) return SFX_ERR_CONFIG;
      if ((rc = expect_f64(hs[0], "A", err)) || (rc = expect_f64(hs[1], "B", err)) || (rc = expect_f64(hs[2], "C", err)))
        return rc;
      const bool tb = d.iparam[0] != 0;
      const int64_t M = hs[0]->rows, K = hs[0]->cols;
      const int64_t bk = tb ? hs[1]->cols : hs[1]->rows, N = tb ? hs[1]->rows : hs[1]->cols;
      if (bk != K || hs[2]->rows != M || hs[2]->cols != N) {
        err = fmt("dgemm shapes do not conform: A %lldx%lld, B %lldx%lld%s, C %lldx%lld", (long long)M, (long long)K,
                  (long long)hs[1]->rows, (long long)hs[1]->cols, tb ? "^T" : "", (long long)hs[2]->rows,
                  (long long)hs[2]->cols);
        return SFX_ERR_CONFIG;
      }
      return 0;
    }
    case SFX_OP_DSYRK:
      if (!need(2) || !writes(1)) return SFX_ERR_CONFIG;
      if ((rc = expect_f64(hs[0], "A", err)) || (rc = expect_f64(hs[1], "C", err))) return rc;
      if (hs[1]->rows != hs[1]->cols || hs[1]->rows != hs[0]->rows) {
        err = "dsyrk: C must be square with A's row count";
        return SFX_ERR_CONFIG;
      }
      return 0;
    case SFX_OP_DTRSM:
      if (!need(2) || !writes(1)) return SFX_ERR_CONFIG;
      if ((rc = expect_f64(hs[0], "L", err)) || (rc = expect_f64(hs[1], "B", err))) return rc;
      if (hs[0]->rows != hs[0]->cols || hs[1]->cols != hs[0]->rows) {
        err = "dtrsm: L must be square with B's column count";
        return SFX_ERR_CONFIG;
      }
      if (d.iparam[0] == 2 && !fullinv_size(hs[0]->rows)) {
        err = "dtrsm (full inverse): L must be 64 * 2^k with 128 <= n <= 2048";
        return SFX_ERR_CONFIG;
      }
      return 0;
    case SFX_OP_DPOTRF:
      if (!need(1) || !writes(0)) return SFX_ERR_CONFIG;
      if ((rc = expect_f64(hs[0], "A", err))) return rc;
      if (hs[0]->rows != hs[0]->cols) {
        err = "dpotrf: A must be square";
        return SFX_ERR_CONFIG;
      }
      if (d.iparam[0] == 2 && !fullinv_size(hs[0]->rows)) {
        err = "dpotrf (full inverse): A must be 64 * 2^k with 128 <= n <= 2048";
        return SFX_ERR_CONFIG;
      }
      return 0;
    case SFX_OP_P2P_PAIR:
      if (!need(4) || !writes(2) || !writes(3)) return SFX_ERR_CONFIG;
      for (int k = 0; k < 4; ++k)
        if ((rc = expect_f64(hs[k], "particle block", err))) return rc;
      if (hs[0]->rows != 4 || hs[1]->rows != 4 || hs[2]->rows != 4 || hs[3]->rows != 4 || hs[0]->cols != hs[2]->cols ||
          hs[1]->cols != hs[3]->cols) {
        err = "p2p: positions/accumulators are 4 x n SoA blocks (x,y,z,q / fx,fy,fz,pot)";
        return SFX_ERR_CONFIG;
      }
      return 0;
    case SFX_OP_P2P_SELF:
      if (!need(2) || !writes(1)) return SFX_ERR_CONFIG;
      for (int k = 0; k < 2; ++k)
        if ((rc = expect_f64(hs[k], "particle block", err))) return rc;
      if (hs[0]->rows != 4 || hs[1]->rows != 4 || hs[0]->cols != hs[1]->cols) {
        err = "p2p: positions/accumulators are 4 x n SoA blocks";
        return SFX_ERR_CONFIG;
      }
      return 0;
    case SFX_OP_DACC:
      if (d.n_access < 2 || d.n_access > 8) {
        err = "dacc takes a target plus 1 to 7 addends";
        return SFX_ERR_CONFIG;
      }
      if (!writes(0)) return SFX_ERR_CONFIG;
      for (uint32_t k = 0; k < d.n_access; ++k) {
        if ((rc = expect_f64(hs[k], "dacc operand", err))) return rc;
        if (hs[k]->rows != hs[0]->rows || hs[k]->cols != hs[0]->cols) {
          err = "dacc: operands must have the same rows x cols";
          return SFX_ERR_CONFIG;
        }
      }
      return 0;
    case SFX_OP_FLUSH:
    case SFX_OP_EXTERN:
      if (!need(1)) return SFX_ERR_CONFIG;
      return 0;
    default:
      if (user_op(d.op)) {  // user ops: up to 8 accesses, the launcher validates the rest
        if (d.n_access > 8) {
          err = "a user op takes at most 8 accesses";
          return SFX_ERR_CONFIG;
        }
        return 0;
      }
      err = fmt("unknown op %u", d.op);
      return SFX_ERR_CONFIG;
  }
}

void Runtime::bind(Task* t, Handle* h, uint32_t mode) {
  // handles.py:209-236: join the last slot only if the category groups, matches,
  // and the slot has not been passed yet; otherwise open a new slot.
  const Cat cat = category_of(mode);
  const bool grouping = cat != CAT_X;
  auto& slots = h->slots;
  uint32_t idx;
  if (grouping && !slots.empty() && slots.back().cat == cat && h->active + 1 <= h->slot_end()) {
    idx = h->slot_end() - 1;
  } else {
    slots.push_back(Slot{cat, {}, 0, 0});
    idx = h->slot_end() - 1;
  }
  h->slot(idx).tasks.push_back(t);
  t->acc.push_back(Access{h, mode, idx});
  if (idx != h->active) {
    t->pending += 1;
  } else if (idx > h->slot_base) {
    // The slot is already active: the previous slot's members were released at
    // launch and may still be running on a device -- wait on their end events.
    // (A retired previous slot had finished entirely.)
    for (Task* p : h->slot(idx - 1).tasks)
      if (p->end && !p->end->complete) t->waits.push_back(p->end);
  }
}

int Runtime::submit(uint32_t n, const sfx_task_desc* descs, const sfx_access* acc) {
  if (!ring_mode_ || n > 16) {
    // batched insertion (insert_gemm / insert_cholesky hand over a block row at a
    // time): the inserter binds it itself, outside the executors' threads -- a
    // thousand-task batch drained by an executor would hold up its launches
    std::unique_lock<std::mutex> lk(mu_);
    drain_locked();  // keep submission order
    return submit_bound(n, descs, acc, true);
  }
  // validate on the calling thread; queue the valid prefix
  uint32_t ok = 0;
  size_t nacc = 0;
  int rc = 0;
  for (; ok < n; ++ok) {
    std::string err;
    rc = validate(descs[ok], acc + nacc, err);
    if (rc) {
      last_error = err;
      break;
    }
    nacc += descs[ok].n_access;
  }
  if (ok > 0) {
    {
      std::lock_guard<std::mutex> g(ring_mu_);
      ring_descs_.insert(ring_descs_.end(), descs, descs + ok);
      ring_acc_.insert(ring_acc_.end(), acc, acc + nacc);
    }
    ring_pending_.store(true);
    if (mu_.try_lock()) {  // nobody busy: bind now
      drain_locked();
      mu_.unlock();
    } else if (sleepers_.load() > 0) {  // an executor is going to sleep: make sure it is bound
      std::unique_lock<std::mutex> lk(mu_);
      drain_locked();
    }
  }
  return rc;
}

void Runtime::drain_locked() {
  if (!ring_pending_.load()) return;
  {
    std::lock_guard<std::mutex> g(ring_mu_);
    ring_pending_.store(false);
    ring_descs_spare_.swap(ring_descs_);
    ring_acc_spare_.swap(ring_acc_);
  }
  if (!ring_descs_spare_.empty()) {
    const int rc = submit_bound(static_cast<uint32_t>(ring_descs_spare_.size()), ring_descs_spare_.data(),
                                ring_acc_spare_.data(), false);
    if (rc) poison(rc, "queued submission: " + last_error);
  }
  ring_descs_spare_.clear();
  ring_acc_spare_.clear();
}

int Runtime::submit_bound(uint32_t n, const sfx_task_desc* descs, const sfx_access* acc, bool check) {
  size_t ai = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const sfx_task_desc& d = descs[i];
    if (check) {
      std::string err;
      const int rc = validate(d, acc + ai, err);
      if (rc) {
        last_error = err;
        return rc;
      }
    }
    if (tasks_by_tid_.count(d.tid)) {
      last_error = fmt("task id %llu reused", (unsigned long long)d.tid);
      return SFX_ERR_INTERNAL;
    }
    Task* t = new_task();
    t->tid = d.tid;
    max_tid_ = std::max(max_tid_, d.tid);
    t->gid = d.graph;
    t->op = d.op;
    t->prio = d.priority;
    t->hint = d.device;
    for (int k = 0; k < 4; ++k) {
      t->fp[k] = d.fparam[k];
      t->ip[k] = d.iparam[k];
    }
    t->acc.reserve(d.n_access);
    for (uint32_t k = 0; k < d.n_access; ++k) bind(t, handles_[acc[ai + k].hid], acc[ai + k].mode);
    t->slot_refs = d.n_access;
    ai += d.n_access;
    // guards: commutative handles (exclusive, or shared for ops that accumulate with
    // device atomics); with several devices also atomic handles, in shared mode:
    // atomic members of one slot run concurrently only on ONE device -- members
    // placed elsewhere wait for them to complete and then pull the result (a
    // serial order of atomic updates is one the atomic semantics allow)
    std::vector<std::pair<Handle*, uint8_t>> guards;
    for (auto& a : t->acc) {
      if (a.mode == SFX_COMMUTATIVE_WRITE)
        guards.emplace_back(a.h, shared_accum(t->op) ? 1 : 0);
      else if (a.mode == SFX_ATOMIC_WRITE && ndev_ > 1)
        guards.emplace_back(a.h, 1);
    }
    std::sort(guards.begin(), guards.end(), [](const auto& x, const auto& y) { return x.first->hid < y.first->hid; });
    for (auto& gp : guards) {
      t->commute.push_back(gp.first);
      t->commute_sh.push_back(gp.second);
    }
    Graph* g = graphs_[d.graph].get();
    g->inserted += 1;
    tasks_by_tid_.put(t->tid, t);
    if (--t->pending == 0) {  // drop the insertion guard (graph.py:161-163)
      t->state = SFX_STATE_READY;
      push_ready(t, -1);
    }
  }
  return SFX_OK;
}

int Runtime::flush(uint32_t gid, uint64_t tid, uint64_t hid, int write_mode) {
  sfx_task_desc d;
  memset(&d, 0, sizeof d);
  d.tid = tid;
  d.graph = gid;
  d.op = SFX_OP_FLUSH;
  d.priority = flush_priority_;
  d.device = -1;
  d.n_access = 1;
  d.iparam[0] = write_mode;
  sfx_access a;
  a.hid = hid;
  a.mode = write_mode ? SFX_WRITE : SFX_READ;
  a.reserved = 0;
  return submit(1, &d, &a);
}

// ------------------------------------------------------------ scheduling

int Runtime::place(Task* t) {
  if (ndev_ == 1) return 0;
  if (t->op == SFX_OP_FLUSH || t->op == SFX_OP_EXTERN) {
    Handle* h = t->acc[0].h;
    if (h->dirty_dev >= 0) return h->dirty_dev;
    for (int e = 0; e < ndev_; ++e)
      if (h->blocks[e] && h->blocks[e]->valid) return e;
    return 0;
  }
  auto grouped = [](uint32_t m) { return m == SFX_ATOMIC_WRITE || m == SFX_COMMUTATIVE_WRITE; };
  int chosen = -1;
  // members of an active atomic/commutative group follow the group's device (it
  // overrides a hint): concurrent members must share one device copy.  Members
  // that still end up elsewhere (a task joining two groups on different devices)
  // are serialised by the shared guards of acquire_commute.
  for (auto& a : t->acc)
    if (grouped(a.mode) && a.h->group_dev >= 0) {
      chosen = a.h->group_dev;
      break;
    }
  if (chosen < 0 && t->hint >= 0) chosen = t->hint % ndev_;
  // owner computes: the device holding the freshest copy of a written tile
  if (chosen < 0)
    for (auto& a : t->acc)
      if (mode_writes(a.mode) && a.h->dirty_dev >= 0) {
        chosen = a.h->dirty_dev;
        break;
      }
  if (chosen < 0)
    for (auto& a : t->acc)
      if (mode_writes(a.mode) && a.h->home >= 0) {
        chosen = a.h->home;
        break;
      }
  if (chosen < 0) {
    // most operand bytes already valid on the device; ties -> least loaded
    uint64_t best_bytes = 0;
    size_t best_load = SIZE_MAX;
    for (int e = 0; e < ndev_; ++e) {
      uint64_t bytes = 0;
      for (auto& a : t->acc)
        if (a.h->blocks[e] && a.h->blocks[e]->valid) bytes += a.h->bytes;
      size_t load = devs_[e]->queue.size() + devs_[e]->ninflight;
      if (chosen < 0 || bytes > best_bytes || (bytes == best_bytes && load < best_load)) {
        chosen = e;
        best_bytes = bytes;
        best_load = load;
      }
    }
  }
  for (auto& a : t->acc)
    if (grouped(a.mode) && a.h->group_dev < 0) a.h->group_dev = chosen;
  return chosen;
}

void Runtime::record(Graph* g, int kind, int64_t t, int wid, uint64_t tid, int64_t extra) {
  if (!trace_ || !g || !g->trace) return;
  sfx_event e;
  e.t_ns = t;
  e.tid = tid;
  e.kind = kind;
  e.worker = wid;
  e.extra = extra;
  g->events.push_back(e);
}

void Runtime::push_ready(Task* t, int wid) {
  // engine.py:212-223: record Push before the task becomes poppable.  A member
  // handed its commutative guards by a release keeps the device it holds them on.
  const int d = (t->guards_held && t->dev >= 0) ? t->dev : place(t);
  t->dev = d;
  t->seq = push_seq_++;
  t->t_push = now_ns();
  record(graphs_[t->gid].get(), SFX_EV_PUSH, t->t_push, wid, t->tid);
  devs_[d]->queue.push(t);
  devs_[d]->prefetch_pending = true;
  devs_[d]->wake_exec();
}

void Runtime::advance(Handle* h) {
  // handles.py:331-343; members of the next slot inherit the finished slot's
  // end events as stream waits
  const uint32_t prev = h->active;
  h->active += 1;
  h->group_dev = -1;
  if (h->graph && !h->graph->history) retire_pending_.push_back(h);
  if (h->active >= h->slot_end()) return;
  Slot& nx = h->slot(h->active);
  const Slot& pv = h->slot(prev);
  for (Task* m : nx.tasks) {
    for (Task* p : pv.tasks)
      if (p->end && !p->end->complete) m->waits.push_back(p->end);
    if (--m->pending == 0) {
      m->state = SFX_STATE_READY;
      push_ready(m, -1);
    }
  }
}

void Runtime::release(Task* t) {
  // handles.py:274-312 (no commutative re-offer: members are chained on events)
  if (t->released) {
    poison(SFX_ERR_INTERNAL, fmt("double release of task %llu", (unsigned long long)t->tid));
    return;
  }
  t->released = true;
  for (auto& a : t->acc) {
    Handle* h = a.h;
    Slot& s = h->slot(a.slot);
    s.done += 1;
    if (a.slot == h->active && s.done >= s.tasks.size()) advance(h);
  }
  flush_retire();
}

// ------------------------------------------------------------ retirement

Task* Runtime::new_task() {
  live_tasks_ += 1;
  if (!task_free_.empty()) {
    Task* t = task_free_.back();
    task_free_.pop_back();
    return t;
  }
  task_store_.push_back(std::make_unique<Task>());
  return task_store_.back().get();
}

void Runtime::free_task(Task* t) {
  tasks_by_tid_.erase(t->tid);
  *t = Task();
  task_free_.push_back(t);
  live_tasks_ -= 1;
  retired_tasks_ += 1;
}

void Runtime::flush_retire() {
  // history-free graphs: pop every slot that is passed (index < active) and whose
  // members all completed; a task goes back to the pool once all its slots went.
  // Runs only at the end of release()/complete(), never while a caller still
  // iterates a task's accesses.
  while (!retire_pending_.empty()) {
    Handle* h = retire_pending_.back();
    retire_pending_.pop_back();
    while (!h->slots.empty() && h->slot_base < h->active) {
      Slot& s = h->slots.front();
      if (s.finished < s.tasks.size()) break;
      for (Task* t : s.tasks)
        if (--t->slot_refs == 0) free_task(t);
      h->slots.pop_front();
      h->slot_base += 1;
    }
  }
}

// --------------------------------------------------------------- arenas

bool Runtime::alloc_space(int d, uint64_t size, uint64_t* off) {
  Device& D = *devs_[d];
  for (auto it = D.free_list.begin(); it != D.free_list.end(); ++it) {
    if (it->second >= size) {
      *off = it->first;
      const uint64_t rest = it->second - size;
      const uint64_t noff = it->first + size;
      D.free_list.erase(it);
      if (rest) D.free_list[noff] = rest;
      D.free_bytes -= size;
      D.stats.bytes_in_use += size;
      return true;
    }
  }
  return false;
}

void Runtime::free_space(int d, uint64_t off, uint64_t size) {
  Device& D = *devs_[d];
  auto it = D.free_list.emplace(off, size).first;
  if (it != D.free_list.begin()) {
    auto pv = std::prev(it);
    if (pv->first + pv->second == it->first) {
      pv->second += it->second;
      D.free_list.erase(it);
      it = pv;
    }
  }
  auto nx = std::next(it);
  if (nx != D.free_list.end() && it->first + it->second == nx->first) {
    it->second += nx->second;
    D.free_list.erase(nx);
  }
  D.free_bytes += size;
  D.stats.bytes_in_use -= size;
}

SyncP Runtime::new_sync(int d, int s, bool timing) {
  auto p = std::make_shared<Sync>();
  p->be = be_;
  p->dev = d;
  p->stream = s;
  p->timing = timing;
  p->event = be_->event_create(d, timing);
  return p;
}

static bool debug_staging() {
  static const bool on = getenv("SFX_DEBUG_STAGING") != nullptr;
  return on;
}

void Runtime::drop_block(Block* b, bool write_back, std::vector<Action>* acts, int s) {
  // device.py:226-232 (+ the write-back leg of evict_victims)
  Handle* h = b->h;
  Device& D = *devs_[b->dev];
  if (b->dirty && write_back && acts) {
    if (b->ready && !b->ready->complete) acts->push_back(Action{Action::WAIT, b->ready});
    Action cp{Action::D2H, nullptr};
    cp.host = h->host;
    cp.src_off = b->off;
    cp.n = h->bytes;
    acts->push_back(cp);
    SyncP hs = new_sync(b->dev, s, false);
    acts->push_back(Action{Action::RECORD, hs});
    h->host_ready = hs;
    h->host_valid = true;
    // the space is reusable below, but the copy above has not read it yet: whoever
    // gets these bytes next waits for the write-back (stream-ordered only on s)
    D.pending_wb.push_back(Device::PendingWriteBack{b->off, b->size, hs});
    if (debug_staging())
      fprintf(stderr, "[sfx] writeback hid=%llu off=%llu stream=%d wait_ready=%d\n", (unsigned long long)h->hid,
              (unsigned long long)b->off, s, (b->ready && !b->ready->complete) ? 1 : 0);
    D.stats.bytes_from_device += h->bytes;
    D.stats.copies_from_device += 1;
    D.stats.writebacks += 1;
  }
  if (h->dirty_dev == b->dev) h->dirty_dev = -1;
  if (b->prefetched) {
    b->prefetched = false;
    b->pins -= 1;
    // its H2D copy may still be in flight on the prefetch stream: the space is only
    // reusable after it (same mechanism as a pending write-back)
    if (b->ready && !b->ready->complete) D.pending_wb.push_back(Device::PendingWriteBack{b->off, b->size, b->ready});
  }
  b->valid = false;
  b->dirty = false;
  h->blocks[b->dev] = nullptr;
  D.blocks.erase(h->hid);
  D.stats.blocks -= 1;
  if (b->pins > 0) {
    b->zombie = true;  // freed when its last in-flight user completes
  } else {
    free_space(b->dev, b->off, b->size);
    b->ready.reset();
    delete b;
  }
}

void Runtime::wait_pending_wb(int d, int s, uint64_t off, uint64_t size, std::vector<Action>& acts) {
  Device& D = *devs_[d];
  size_t keep = 0;
  for (size_t k = 0; k < D.pending_wb.size(); ++k) {
    auto& p = D.pending_wb[k];
    const bool recorded = p.done->recorded.load(std::memory_order_acquire);
    if (recorded && be_->event_done(d, p.done->event)) continue;  // drop finished write-backs
    // a write-back planned on this same stream (possibly in this very plan, not yet
    // recorded) is ordered before our copies by the stream itself
    const bool same_stream = p.done->dev == d && p.done->stream == s;
    if (!same_stream && p.off < off + size && off < p.off + p.size) acts.push_back(Action{Action::WAIT, p.done});
    D.pending_wb[keep++] = p;
  }
  D.pending_wb.resize(keep);
}

int Runtime::evict_one(int d, int s, std::vector<Action>& acts, std::string& err) {
  // device.py:208-224: victim = least (stamp, hid) among unpinned blocks
  Device& D = *devs_[d];
  Block* victim = nullptr;
  for (auto& kv : D.blocks) {
    Block* b = kv.second;
    if (b->pins) continue;
    if (!victim || b->stamp < victim->stamp || (b->stamp == victim->stamp && b->h->hid < victim->h->hid)) victim = b;
  }
  if (!victim) {
    // only blocks held by the prefetcher remain: give one back (clean data, the host
    // copy is valid) rather than waiting for a task that may need that very space
    for (auto& kv : D.blocks) {
      Block* b = kv.second;
      if (!(b->prefetched && b->pins == 1)) continue;
      if (!victim || b->stamp < victim->stamp || (b->stamp == victim->stamp && b->h->hid < victim->h->hid))
        victim = b;
    }
  }
  if (!victim) return 1;
  D.stats.evictions += 1;
  if (debug_staging())
    fprintf(stderr, "[sfx] evict hid=%llu off=%llu dirty=%d stream=%d\n", (unsigned long long)victim->h->hid,
            (unsigned long long)victim->off, victim->dirty ? 1 : 0, s);
  drop_block(victim, true, &acts, s);
  return 0;
}

int Runtime::ensure_block(int d, int s, Handle* h, std::vector<Action>& acts, std::vector<Block*>& tmp_pins,
                          Block** out, std::string& err) {
  // device.py:234-264
  Device& D = *devs_[d];
  const uint64_t size = std::max<uint64_t>((h->bytes + align_ - 1) / align_ * align_, align_);
  if (size > D.capacity) {
    err = fmt("device %d: object of %llu bytes exceeds the %llu-byte arena", d, (unsigned long long)h->bytes,
              (unsigned long long)D.capacity);
    return SFX_ERR_STAGING;
  }
  Block* b = h->blocks[d];
  if (!b) {
    auto pinned_by_others = [&]() {
      size_t mine = 0, all = 0;
      for (auto& kv : D.blocks)
        if (!(kv.second->prefetched && kv.second->pins == 1)) all += kv.second->pins;  // prefetch pins yield
      for (Block* p : tmp_pins)
        if (p->dev == d) mine += 1;
      if (all > mine) return true;
      // blocks pinned by tasks of OTHER devices (peer-pull sources) -- and zombies
      // (invalidated while pinned, already out of D.blocks) -- are released by
      // completions anywhere: wait while any device has work in flight
      for (auto& dv : devs_)
        if (dv->ninflight > 0) return true;
      return false;
    };
    while (D.free_bytes < size) {
      if (evict_one(d, s, acts, err)) {
        if (pinned_by_others()) return 1;
        err = fmt("device %d: need %llu bytes but every block is pinned by a running task", d,
                  (unsigned long long)size);
        return SFX_ERR_STAGING;
      }
    }
    uint64_t off;
    while (!alloc_space(d, size, &off)) {
      if (evict_one(d, s, acts, err)) {
        if (pinned_by_others()) return 1;
        err = fmt("device %d: fragmentation and pinned blocks prevent a %llu-byte allocation", d,
                  (unsigned long long)size);
        return SFX_ERR_STAGING;
      }
    }
    wait_pending_wb(d, s, off, size, acts);
    b = new Block();
    b->h = h;
    b->dev = d;
    b->off = off;
    b->size = size;
    h->blocks[d] = b;
    D.blocks[h->hid] = b;
    D.stats.blocks += 1;
  }
  if (b->prefetched)
    b->prefetched = false;  // the prefetch's pin becomes this task's pin
  else
    b->pins += 1;
  tmp_pins.push_back(b);
  *out = b;
  return 0;
}

// ------------------------------------------------------------- execution

int Runtime::plan(int d, int s, Task* t, std::vector<Action>& acts, OpLaunch& op, std::string& err,
                  bool record_start) {
  Device& D = *devs_[d];
  auto wait_on = [&](const SyncP& p) {
    if (!p || p->complete) return;
    if (p->dev == d && p->stream == s) return;  // same stream: ordered
    acts.push_back(Action{Action::WAIT, p});
  };
  // pass 1: blocks for every operand (may evict; victims are written back)
  std::vector<Block*> pins;
  std::vector<Block*> blocks(t->acc.size(), nullptr);
  if (t->op != SFX_OP_FLUSH && t->op != SFX_OP_EXTERN) {
    for (size_t k = 0; k < t->acc.size(); ++k) {
      int rc = ensure_block(d, s, t->acc[k].h, acts, pins, &blocks[k], err);
      if (rc) {
        for (Block* b : pins) {
          if (--b->pins == 0 && b->zombie) {
            free_space(b->dev, b->off, b->size);
            delete b;
          }
        }
        return rc;
      }
    }
  }
  if (!t->end) {
    t->end = new_sync(d, s, ktime_);
    if (ktime_) t->start = new_sync(d, s, true);
  }
  for (const SyncP& w : t->waits) wait_on(w);
  for (auto& a : t->acc)
    if (a.mode == SFX_COMMUTATIVE_WRITE) wait_on(a.h->commute_last);
  if (t->start && record_start) acts.push_back(Action{Action::RECORD, t->start});

  if (t->op == SFX_OP_EXTERN) {
    // make the host buffer current for the agent: a read (send) fetches the dirty
    // copy home and keeps device copies; a write (recv) drops every device copy
    // (the agent overwrites the whole buffer; host_valid is set by extern_done)
    Handle* h = t->acc[0].h;
    if (!mode_writes(t->acc[0].mode)) {
      if (h->dirty_dev >= 0) {
        Block* b = h->blocks[h->dirty_dev];
        if (h->dirty_dev != d) {
          err = "extern task placed away from the dirty copy";
          return SFX_ERR_INTERNAL;
        }
        wait_on(b->ready);
        Action cp{Action::D2H, nullptr};
        cp.host = h->host;
        cp.src_off = b->off;
        cp.n = h->bytes;
        acts.push_back(cp);
        b->dirty = false;
        b->pins += 1;
        t->pinned.push_back(b);
        h->dirty_dev = -1;
        h->host_valid = true;
        h->host_ready = t->end;
        D.stats.bytes_from_device += h->bytes;
        D.stats.copies_from_device += 1;
      } else {
        wait_on(h->host_ready);
      }
    } else {
      for (int e = 0; e < ndev_; ++e)
        if (h->blocks[e]) drop_block(h->blocks[e], false, nullptr, s);
      h->dirty_dev = -1;
      h->host_valid = false;
    }
    op.op = SFX_OP_EXTERN;
    op.n = 0;
    return 0;
  }
  if (t->op == SFX_OP_FLUSH) {
    // graph.py:258-260 + device.py:318-326: fetch the dirty copy home; a
    // write-mode flush then drops every device copy
    Handle* h = t->acc[0].h;
    if (h->dirty_dev >= 0) {
      Block* b = h->blocks[h->dirty_dev];
      if (h->dirty_dev != d) {
        err = "flush placed away from the dirty copy";
        return SFX_ERR_INTERNAL;
      }
      wait_on(b->ready);
      Action cp{Action::D2H, nullptr};
      cp.host = h->host;
      cp.src_off = b->off;
      cp.n = h->bytes;
      acts.push_back(cp);
      b->dirty = false;
      b->pins += 1;
      t->pinned.push_back(b);
      h->dirty_dev = -1;
      h->host_valid = true;
      h->host_ready = t->end;
      D.stats.bytes_from_device += h->bytes;
      D.stats.copies_from_device += 1;
    }
    if (t->ip[0]) {
      for (int e = 0; e < ndev_; ++e)
        if (h->blocks[e]) drop_block(h->blocks[e], false, nullptr, s);
    }
    op.op = SFX_OP_FLUSH;
    op.n = 0;
    return 0;
  }

  // pass 2: make every operand valid on d (device.py:340-369)
  for (size_t k = 0; k < t->acc.size(); ++k) {
    Handle* h = t->acc[k].h;
    Block* b = blocks[k];
    if (b->valid) {
      D.stats.hits += 1;
      wait_on(b->ready);
    } else {
      D.stats.misses += 1;
      int src = -1;
      if (h->dirty_dev >= 0 && h->dirty_dev != d) {
        src = h->dirty_dev;
      } else {
        for (int e = 0; e < ndev_; ++e)
          if (e != d && h->blocks[e] && h->blocks[e]->valid) {
            src = e;
            break;
          }
      }
      // host staging on the copy stream: every H2D of this device in one FIFO
      // (dispatch order = priority order), so the first groups' operands arrive
      // first instead of every stream's copies sharing PCIe until all are done
      const int cs = src < 0 && stage_stream_ ? pf_stream() : -1;
      const int ws = cs >= 0 ? cs : s;
      // the block may have been allocated by an earlier, failed plan over a range
      // whose previous contents are still being written back on another stream:
      // the copy into it must wait for that write-back (allocation-time waits
      // only cover blocks allocated by this plan)
      const size_t a0 = acts.size();
      wait_pending_wb(d, ws, b->off, b->size, acts);
      for (size_t q = a0; q < acts.size(); ++q) acts[q].stream = cs;
      if (src >= 0) {
        Block* sb = h->blocks[src];
        wait_on(sb->ready);
        Action cp{Action::P2P, nullptr};
        cp.src_dev = src;
        cp.src_off = sb->off;
        cp.dst_off = b->off;
        cp.n = h->bytes;
        acts.push_back(cp);
        sb->pins += 1;
        t->pinned.push_back(sb);
        D.stats.bytes_p2p_in += h->bytes;
        D.stats.copies_p2p_in += 1;
      } else {
        if (!h->host_valid) {
          err = fmt("handle %llu has no valid copy anywhere", (unsigned long long)h->hid);
          return SFX_ERR_INTERNAL;
        }
        if (cs < 0) {
          wait_on(h->host_ready);
        } else if (h->host_ready && !h->host_ready->complete && !(h->host_ready->dev == d && h->host_ready->stream == cs)) {
          Action w{Action::WAIT, h->host_ready};
          w.stream = cs;
          acts.push_back(w);
        }
        if (debug_staging())
          fprintf(stderr, "[sfx] stage hid=%llu off=%llu stream=%d task=%llu host_ready=%s\n",
                  (unsigned long long)h->hid, (unsigned long long)b->off, ws, (unsigned long long)t->tid,
                  !h->host_ready ? "none" : (h->host_ready->complete ? "complete" : (h->host_ready->stream == ws ? "same-stream" : "waited")));
        Action cp{Action::H2D, nullptr};
        cp.host = h->host;
        cp.dst_off = b->off;
        cp.n = h->bytes;
        cp.stream = cs;
        acts.push_back(cp);
        D.stats.bytes_to_device += h->bytes;
        D.stats.copies_to_device += 1;
      }
      SyncP csync = new_sync(d, ws, false);
      Action rec{Action::RECORD, csync};
      rec.stream = cs;
      acts.push_back(rec);
      if (cs >= 0) acts.push_back(Action{Action::WAIT, csync});  // the group waits on its copy
      t->copy_syncs.push_back(csync);
      b->valid = true;
      b->ready = csync;
    }
    b->stamp = ++D.clock;
    t->pinned.push_back(b);  // the pass-1 pin is released at completion
  }

  // pass 3: coherency of written operands
  for (size_t k = 0; k < t->acc.size(); ++k) {
    const uint32_t m = t->acc[k].mode;
    if (!mode_writes(m)) continue;
    Handle* h = t->acc[k].h;
    Block* b = blocks[k];
    for (int e = 0; e < ndev_; ++e)
      if (e != d && h->blocks[e]) drop_block(h->blocks[e], false, nullptr, s);  // device.py:298-314
    b->dirty = true;
    h->dirty_dev = d;
    h->host_valid = false;
    if (m == SFX_COMMUTATIVE_WRITE && !shared_accum(t->op)) h->commute_last = t->end;
    if (m == SFX_WRITE || m == SFX_MAYBE_WRITE) b->ready = t->end;
  }

  if (debug_staging()) {
    fprintf(stderr, "[sfx] plan task=%llu op=%u stream=%d", (unsigned long long)t->tid, t->op, s);
    for (size_t k = 0; k < t->acc.size(); ++k)
      fprintf(stderr, " [hid=%llu off=%llu m=%u]", (unsigned long long)t->acc[k].h->hid,
              (unsigned long long)blocks[k]->off, t->acc[k].mode);
    fprintf(stderr, " waits=%zu\n", t->waits.size());
  }
  op.op = t->op;
  op.deterministic = deterministic_;
  op.n = static_cast<int>(std::min<size_t>(t->acc.size(), 8));
  if (t->op == SFX_OP_DPOTRF && t->status_slot < 0) t->status_slot = be_->status_alloc(d);
  op.status_slot = t->status_slot;
  for (int k = 0; k < op.n; ++k) {
    Handle* h = t->acc[k].h;
    op.o[k].dptr = be_->arena_ptr(d, blocks[k]->off);
    op.o[k].bytes = h->bytes;
    op.o[k].rows = h->rows;
    op.o[k].cols = h->cols;
    op.o[k].ld = h->ld;
    op.o[k].dtype = h->dtype;
    op.o[k].mode = t->acc[k].mode;
  }
  for (int k = 0; k < 4; ++k) {
    op.fp[k] = t->fp[k];
    op.ip[k] = t->ip[k];
  }
  return 0;
}

int Runtime::issue(int d, int s, const std::vector<Task*>& group, std::vector<Action>& acts,
                   std::vector<OpLaunch>& ops, std::string& err) {
  int rc = 0;
  const int s_group = s;
  for (Action& a : acts) {
    s = a.stream >= 0 ? a.stream : s_group;
    switch (a.kind) {
      case Action::WAIT: {
        if (debug_staging())
          fprintf(stderr, "[sfx]   issue s=%d WAIT on stream %d%s\n", s, a.sync->stream,
                  (a.sync->dev == d && a.sync->stream == s) ? " (same, skipped)" : "");
        if (a.sync->dev == d && a.sync->stream == s) break;  // stream order suffices
        while (!a.sync->recorded.load(std::memory_order_acquire)) std::this_thread::yield();
        rc = be_->stream_wait(d, s, a.sync->event, err);
        devs_[d]->stats.stream_waits += 1;
        break;
      }
      case Action::H2D:
        if (debug_staging()) fprintf(stderr, "[sfx]   issue s=%d H2D off=%llu\n", s, (unsigned long long)a.dst_off);
        rc = be_->copy_h2d(d, s, a.dst_off, a.host, a.n, err);
        break;
      case Action::D2H:
        if (debug_staging()) fprintf(stderr, "[sfx]   issue s=%d D2H off=%llu\n", s, (unsigned long long)a.src_off);
        rc = be_->copy_d2h(d, s, a.host, a.src_off, a.n, err);
        break;
      case Action::P2P:
        rc = be_->copy_p2p(d, s, a.dst_off, a.src_dev, a.src_off, a.n, err);
        break;
      case Action::RECORD:
        rc = be_->event_record(d, s, a.sync->event, err);
        a.sync->recorded.store(true, std::memory_order_release);
        break;
    }
    if (rc) return rc;
  }
  s = s_group;
  if (group.empty()) return 0;
  std::vector<OpLaunch> kern;
  kern.reserve(ops.size());
  for (auto& op : ops)
    if (op.op != SFX_OP_FLUSH && op.op != SFX_OP_NOOP && op.op != SFX_OP_EXTERN) kern.push_back(op);
  if (!kern.empty()) {
    if (debug_staging()) fprintf(stderr, "[sfx]   issue s=%d launch task=%llu\n", s, (unsigned long long)group[0]->tid);
    rc = be_->launch_group(d, s, kern, err);
    if (rc) return rc;
    devs_[d]->stats.kernel_launches += kern.size();  // sim: ops executed
  }
  SyncP end = group[0]->end;
  rc = be_->event_record(d, s, end->event, err);
  end->recorded.store(true, std::memory_order_release);
  return rc;
}

bool Runtime::is_coop(const Task* t) const {
  if (ncoop_ == 0) return false;
  if (t->op == SFX_OP_DPOTRF) return t->acc[0].h->rows % 64 == 0 && t->acc[0].h->rows <= 4096;
  if (t->op == SFX_OP_DTRSM)  // the inverse-block variant runs as ordinary DMMA GEMM launches
    return !t->ip[0] && t->acc[0].h->rows % 64 == 0 && t->acc[0].h->rows <= 4096 && t->acc[1].h->rows % 64 == 0;
  return false;
}

bool Runtime::groupable(const Task* t) const {
  // only ops with a grouped kernel (one launch for the whole group) or trivial
  // generators: grouping anything else would serialise independent tasks on one stream
  switch (t->op) {
    case SFX_OP_DTRSM:  // grouped cooperative TRSM, or grouped inverse-block GEMM sweeps
      // full inverse: a group is ONE unsplit TRI-masked DGEMM over all its members
      // (a lone TRSM keeps the K-weighted split: lower latency on the panel chain)
      if (t->ip[0] == 2) return group_max_ > 1;
      return group_max_ > 1 && (is_coop(t) || (t->ip[0] && t->acc[0].h->rows % 64 == 0));
    case SFX_OP_DGEMM:
    case SFX_OP_DSYRK:
    case SFX_OP_FILL_UNIFORM:
    case SFX_OP_FILL_SPD:
    case SFX_OP_FILL_PARTICLES:
    case SFX_OP_ZERO:
    case SFX_OP_P2P_PAIR:  // grouped mutual P2P kernel; commutative guards in shared mode
    case SFX_OP_P2P_SELF:
      return group_max_ > 1 && !deterministic_;  // deterministic: one-sided kernel per task
    case SFX_OP_NOOP:  // no device work: ready empty tasks share one end event (one record per group)
      return group_max_ > 1;
    case SFX_OP_SPIN:  // same-duration spins: one CTA per member in one launch, all concurrent
      return group_max_ > 1 && !be_->is_sim();  // (the simulated backend would run them one by one)
    default:
      return false;
  }
}

bool Runtime::same_signature(const Task* a, const Task* b) const {
  if (a->op != b->op || a->acc.size() != b->acc.size()) return false;
  const bool ip_matters =
      a->op == SFX_OP_DGEMM || a->op == SFX_OP_DTRSM || a->op == SFX_OP_DPOTRF || a->op == SFX_OP_SPIN;
  for (int k = 0; k < 4; ++k)
    if (a->fp[k] != b->fp[k] || (ip_matters && a->ip[k] != b->ip[k])) return false;
  for (size_t k = 0; k < a->acc.size(); ++k) {
    const Handle* x = a->acc[k].h;
    const Handle* y = b->acc[k].h;
    if (x->rows != y->rows || x->cols != y->cols || x->ld != y->ld || x->dtype != y->dtype ||
        a->acc[k].mode != b->acc[k].mode)
      return false;
  }
  return true;
}

bool Runtime::acquire_commute(Task* t) {
  // all-or-nothing in hid order; on failure the task parks on the busy handle.
  // Shared mode (the op accumulates into the handle with device atomics, or an
  // atomic_write access, so any interleaving is one of the orders the semantics
  // allow): members run concurrently as long as they are on the same device and
  // no exclusive member holds the handle.
  if (t->guards_held) return true;  // acquired when a release handed the handle over
  for (size_t k = 0; k < t->commute.size(); ++k) {
    Handle* h = t->commute[k];
    const bool busy = t->commute_sh[k]
                          ? (h->commute_owner != nullptr || (h->shared_users > 0 && h->shared_dev != t->dev))
                          : ((h->commute_owner && h->commute_owner != t) || h->shared_users > 0);
    if (busy) {
      h->commute_waiters.push_back(t);
      return false;
    }
  }
  for (size_t k = 0; k < t->commute.size(); ++k) {
    Handle* h = t->commute[k];
    if (t->commute_sh[k]) {
      h->shared_users += 1;
      h->shared_dev = t->dev;
    } else {
      h->commute_owner = t;
    }
  }
  t->guards_held = true;
  return true;
}

static bool exclusive_guards(const Task* t) {
  for (size_t k = 0; k < t->commute.size(); ++k)
    if (t->commute_sh[k]) return false;
  return true;
}

static bool shared_on(const Task* t, const Handle* h) {
  for (size_t k = 0; k < t->commute.size(); ++k)
    if (t->commute[k] == h) return t->commute_sh[k] != 0;
  return false;
}

void Runtime::release_commute(Task* t) {
  if (!t->guards_held) return;
  t->guards_held = false;
  for (size_t k = 0; k < t->commute.size(); ++k) {
    Handle* h = t->commute[k];
    if (t->commute_sh[k]) {
      if (--h->shared_users > 0) continue;
      h->shared_dev = -1;
    } else {
      if (h->commute_owner != t) continue;
      h->commute_owner = nullptr;
    }
    // hand the freed handle to the parked members in FIFO order: each is tried
    // right here (all-or-nothing over all its handles) and only a winner re-enters
    // its device queue; a member that still finds another handle busy re-parks on
    // that one.  Every waiter is touched O(1) times per handle it waits on -- not
    // re-offered on every release (the reference's quadratic re-offer,
    // handles.py:317-328).  Exclusive: the first winner owns h, the rest stay
    // parked.  Shared: winners on h's new device keep coming until one parks on h.
    size_t budget = h->commute_waiters.size();
    while (budget-- > 0 && !h->commute_waiters.empty()) {
      Task* w = h->commute_waiters.front();
      h->commute_waiters.pop_front();
      if (acquire_commute(w)) {
        push_ready(w, -1);
        if (!shared_on(w, h)) break;
        continue;
      }
      if (!h->commute_waiters.empty() && h->commute_waiters.back() == w) break;  // h itself is taken again
    }
  }
}

bool Runtime::commute_conflict(const std::vector<Task*>& group, const Task* t) const {
  // members of one commutative group must never run concurrently on the same
  // handle -- unless both take it in shared mode
  for (size_t k = 0; k < t->commute.size(); ++k) {
    const Handle* h = t->commute[k];
    for (const Task* g : group)
      for (size_t j = 0; j < g->commute.size(); ++j)
        if (g->commute[j] == h && !(t->commute_sh[k] && g->commute_sh[j])) return true;
  }
  return false;
}

void Runtime::complete(Task* t) {
  Device& D = *devs_[t->dev];
  if (!t->detached && t->end && !t->end->group_counted) {
    t->end->group_counted = true;
    D.stream_groups[t->stream] -= 1;
    D.stage_inflight -= t->end->staged;
  }
  if (t->end) t->end->complete = true;
  if (t->start) t->start->complete = true;
  for (auto& c : t->copy_syncs) c->complete = true;
  for (Block* b : t->pinned) {
    if (--b->pins == 0 && b->zombie) {
      free_space(b->dev, b->off, b->size);
      b->ready.reset();
      delete b;
    }
  }
  t->pinned.clear();
  t->copy_syncs.clear();
  t->waits.clear();
  if (t->status_slot >= 0) {
    // engine.py:227-243: a failing body poisons the engine; the cause names the task
    const int info = be_->status_take(t->dev, t->status_slot);
    t->status_slot = -1;
    if (info != 0)
      poison(SFX_ERR_NUMERIC, fmt("dpotrf (task %llu): the leading minor of order %d is not positive definite",
                                  (unsigned long long)t->tid, info));
  }
  Graph* g = graphs_[t->gid].get();
  auto when = [&](Sync* sy) { return sy->t_resolved ? sy->t_ns : be_->event_time_ns(t->dev, sy->event); };
  if (ktime_ && t->start && t->end) {
    D.stats.timed_tasks += 1;
    if (!t->end->group_timed) {
      t->end->group_timed = true;
      const int64_t t0 = when(t->start.get());
      const int64_t t1 = when(t->end.get());
      const int64_t dt = t1 - t0;
      if (dt > 0) D.kintervals.emplace_back(t0, t1);
      D.stats.timed_groups += 1;
      D.stats.timed_ns += dt > 0 ? static_cast<uint64_t>(dt) : 0;
    }
  }
  if (trace_ && t->end && (t->start || t->op == SFX_OP_NOOP)) {
    t->t_end = when(t->end.get());
    t->t_start = t->start ? when(t->start.get()) : t->t_end;
    const int wid = t->dev * (nstreams_ + nurgent_ + ncoop_) + t->stream;
    record(g, SFX_EV_START, t->t_start, wid, t->tid);
    record(g, SFX_EV_END, t->t_end, wid, t->tid);
  }
  t->start.reset();
  t->end.reset();
  t->state = SFX_STATE_FINISHED;
  if (!t->commute.empty()) release_commute(t);
  g->completed += 1;
  if (!t->detached) {
    D.ninflight -= 1;
    D.stream_inflight[t->stream] -= 1;
  }
  D.stats.tasks_executed += 1;
  D.wake_exec();
  done_cv_.notify_all();
  if (!g->history) {
    for (auto& a : t->acc) {
      a.h->slot(a.slot).finished += 1;
      retire_pending_.push_back(a.h);
    }
    flush_retire();  // may free t: nothing below touches it
  }
}

void Runtime::extern_handoff(Task* t) {
  // the stream slot is free as soon as the host copy is current: a recv may wait
  // for its peer for a long time
  Device& D = *devs_[t->dev];
  if (t->end && !t->end->group_counted) {
    t->end->group_counted = true;
    D.stream_groups[t->stream] -= 1;
    D.stage_inflight -= t->end->staged;
  }
  D.ninflight -= 1;
  D.stream_inflight[t->stream] -= 1;
  t->detached = true;
  extern_ready_.push_back(t);
  extern_cv_.notify_all();
  D.wake_exec();
}

int Runtime::extern_poll(uint64_t* tids, uint64_t cap, uint64_t* n, double timeout_s) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  auto ready = [&] { return stopping_ || fail_code_ != 0 || !extern_ready_.empty(); };
  if (timeout_s < 0)
    extern_cv_.wait(lk, ready);
  else
    extern_cv_.wait_for(lk, std::chrono::duration<double>(timeout_s), ready);
  uint64_t k = 0;
  while (k < cap && !extern_ready_.empty()) {
    tids[k++] = extern_ready_.front()->tid;
    extern_ready_.pop_front();
  }
  *n = k;
  return SFX_OK;
}

int Runtime::extern_done(uint64_t tid, int status, const char* msg) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  Task* t = tasks_by_tid_.get(tid);
  if (!t || t->op != SFX_OP_EXTERN || !t->detached) {
    last_error = "extern_done: not an external task handed out by sfx_extern_poll";
    return SFX_ERR_CONFIG;
  }
  if (status != 0) {
    poison(SFX_ERR_ENGINE_FAILED, msg ? msg : "external task failed");
    return SFX_OK;
  }
  Handle* h = t->acc[0].h;
  if (mode_writes(t->acc[0].mode)) {  // the agent wrote the host buffer
    h->host_valid = true;
    h->host_ready.reset();
    h->dirty_dev = -1;
  }
  release(t);
  complete(t);
  return SFX_OK;
}

int Runtime::fail(const std::string& msg) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  poison(SFX_ERR_ENGINE_FAILED, msg);
  return SFX_OK;
}

void Runtime::poison(int code, const std::string& msg) {
  // engine.py:227-243: first failure wins; everyone waiting learns of it
  if (!fail_code_) {
    fail_code_ = code;
    fail_msg_ = msg;
  }
  extern_cv_.notify_all();
  for (auto& d : devs_) {
    d->exec_cv.notify_all();
    d->comp_cv.notify_all();
  }
  done_cv_.notify_all();
}

int Runtime::plan_prefetch(int d, std::vector<Action>& acts) {
  Device& D = *devs_[d];
  const int s = pf_stream();
  int issued = 0, seen = 0;
  auto consider = [&](Task* t) {
    if (t->op == SFX_OP_FLUSH) return;
    for (auto& a : t->acc) {
      Handle* h = a.h;
      if (h->blocks[d] || !h->host_valid || h->dirty_dev >= 0) continue;
      const uint64_t size = std::max<uint64_t>((h->bytes + align_ - 1) / align_ * align_, align_);
      if (D.free_bytes < size + D.capacity / 8) return;
      uint64_t off;
      if (!alloc_space(d, size, &off)) return;
      wait_pending_wb(d, s, off, size, acts);
      Block* b = new Block();
      b->h = h;
      b->dev = d;
      b->off = off;
      b->size = size;
      b->pins = 1;
      b->prefetched = true;
      b->valid = true;
      b->stamp = ++D.clock;
      h->blocks[d] = b;
      D.blocks[h->hid] = b;
      D.stats.blocks += 1;
      if (h->host_ready && !h->host_ready->complete) acts.push_back(Action{Action::WAIT, h->host_ready});
      Action cp{Action::H2D, nullptr};
      cp.host = h->host;
      cp.dst_off = off;
      cp.n = h->bytes;
      acts.push_back(cp);
      if (debug_staging())
        fprintf(stderr, "[sfx] prefetch hid=%llu off=%llu stream=%d\n", (unsigned long long)h->hid,
                (unsigned long long)off, s);
      SyncP cs = new_sync(d, s, false);
      acts.push_back(Action{Action::RECORD, cs});
      b->ready = cs;
      D.stats.bytes_to_device += h->bytes;
      D.stats.copies_to_device += 1;
      D.stats.prefetches += 1;
      ++issued;
    }
  };
  if (!D.queue.prio) {
    for (Task* t : D.queue.fifo) {
      if (++seen > prefetch_depth_) break;
      consider(t);
    }
  } else {
    std::vector<Task*> top(D.queue.heap);
    std::sort(top.begin(), top.end(), [](const Task* a, const Task* b) { return heap_less(b, a); });
    for (Task* t : top) {
      if (++seen > prefetch_depth_) break;
      consider(t);
    }
  }
  return issued;
}

void Runtime::exec_loop(int d) {
  be_->bind_thread(d);
  Device& D = *devs_[d];
  std::unique_lock<std::mutex> lk(mu_);
  std::vector<Task*> group;
  std::vector<Action> acts;
  std::vector<OpLaunch> ops;
  while (true) {
    auto free_in = [&](int lo, int hi) {
      int best = -1;
      for (int k = lo; k < hi; ++k)
        if (D.stream_groups[k] < static_cast<int>(groups_per_stream_) &&
            (best < 0 || D.stream_inflight[k] < D.stream_inflight[best]))
          best = k;
      return best;
    };
    // Stream affinity: a task whose predecessor is still in flight on a stream of
    // its class joins that stream (ordered by the stream itself, no event wait).
    // Otherwise a chain's successor can queue behind ANOTHER chain's task on a
    // shared stream and inherit its wait (head-of-line blocking: the reference
    // overhead protocol, T chains of 1 ms tasks, ran at 2 ms per chain step).
    auto affine = [&](const Task* t, int lo, int hi) {
      if (!stream_affinity_) return -1;
      for (const SyncP& w : t->waits)
        if (w && !w->complete && w->dev == d && w->stream >= lo && w->stream < hi &&
            D.stream_groups[w->stream] < static_cast<int>(groups_per_stream_))
          return w->stream;
      return -1;
    };
    auto pick = [&](const Task* t, int lo, int hi) {
      const int s = affine(t, lo, hi);
      return s >= 0 ? s : free_in(lo, hi);
    };
    // urgent tasks prefer the high-priority streams and may fall back to normal
    // ones; normal tasks never take an urgent stream
    auto free_stream = [&](const Task* t) {
      if (is_coop(t)) return free_in(nstreams_ + nurgent_, nstreams_ + nurgent_ + ncoop_);
      if (nurgent_ > 0 && t->prio >= urgent_priority_) {
        int s = pick(t, nstreams_, nstreams_ + nurgent_);
        return s >= 0 ? s : pick(t, 0, nstreams_);
      }
      return pick(t, 0, nstreams_);
    };
    auto staging_bytes = [&](const Task* t) {
      uint64_t n = 0;
      for (const Access& a : t->acc)
        if (!a.h->blocks[d]) n += std::max<uint64_t>((a.h->bytes + align_ - 1) / align_ * align_, align_);
      return n;
    };
    auto stage_ok = [&] {
      return !stage_window_ || D.stage_inflight == 0 ||
             D.stage_inflight + staging_bytes(D.queue.peek()) <= stage_window_;
    };
    auto runnable = [&] {
      return !paused_ && !fail_code_ && D.queue.size() > 0 && D.ninflight < static_cast<int>(window_) &&
             free_stream(D.queue.peek()) >= 0 && stage_ok();
    };
    drain_locked();  // submissions queued while mu_ was busy
    while (!(stopping_ || runnable() || (prefetch_ && D.prefetch_pending && !paused_ && !fail_code_))) {
      D.exec_sleeping = true;
      sleepers_.fetch_add(1);
      if (ring_pending_.load()) {  // queued after the drain above: bind them instead of sleeping
        sleepers_.fetch_sub(1);
        D.exec_sleeping = false;
        drain_locked();
        continue;
      }
      D.exec_cv.wait(lk);
      sleepers_.fetch_sub(1);
      D.exec_sleeping = false;
    }
    if (stopping_) return;
    if (!runnable()) {
      // every stream is busy: stage operands of queued tasks meanwhile
      D.prefetch_pending = false;
      std::vector<Action> pacts;
      if (plan_prefetch(d, pacts) > 0) {
        lk.unlock();
        std::string perr;
        std::vector<Task*> none;
        std::vector<OpLaunch> noops;
        int prc = issue(d, pf_stream(), none, pacts, noops, perr);
        lk.lock();
        if (prc) poison(SFX_ERR_CUDA, perr);
      }
      continue;
    }
    const int64_t t_busy0 = now_ns();
    // pop the head task, plus (grouped launch) the following ready tasks of the
    // same op and operand shapes -- up to group_max_, never two commutative
    // members of one handle
    group.clear();
    Task* first = D.queue.pop();
    if (!first->commute.empty() && !acquire_commute(first)) continue;  // parked until the guard frees
    group.push_back(first);
    // A group only grows while the operands its members still have to stage fit in
    // the free arena space, so no member evicts between the members of one
    // launch: under a tile cache much smaller than the working set this cuts the
    // eviction traffic (C3 with a 3 GiB arena: 25.9 -> 27.3 TFLOP/s).  (It first
    // served as the mitigation of the write-back race fixed in plan() pass 2; with
    // SFX_GROUP_NO_STAGE_LIMIT=1 the limit is off, tools/arena_stress.py stays correct.)
    static const bool no_stage_limit = getenv("SFX_GROUP_NO_STAGE_LIMIT") != nullptr;  // for stress tests
    uint64_t group_stage = staging_bytes(first);
    if (groupable(first) && (no_stage_limit || group_stage <= D.free_bytes)) {
      const bool urgent = first->prio >= urgent_priority_;
      while (group.size() < group_max_ && D.queue.size() > 0 &&
             D.ninflight + static_cast<int>(group.size()) < static_cast<int>(window_)) {
        Task* nx = D.queue.peek();
        if (!same_signature(first, nx) || commute_conflict(group, nx) || (nx->prio >= urgent_priority_) != urgent)
          break;
        if (first->op == SFX_OP_DTRSM && nx->prio != first->prio) break;  // a critical TRSM launches alone
        const uint64_t more = staging_bytes(nx);
        if (!no_stage_limit && group_stage + more > D.free_bytes) break;  // would evict mid-group
        group_stage += more;
        D.queue.pop();
        if (!nx->commute.empty() && !acquire_commute(nx)) continue;
        group.push_back(nx);
      }
    }
    const int s = free_stream(first);
    SyncP gend = new_sync(d, s, ktime_);
    // a group of empty tasks (noop: no kernel) starts where it ends -- one timing
    // event instead of two (timing event records dominated the per-task cost of
    // the reference overhead protocol at D = 0 with tracing on)
    const bool empty_group = first->op == SFX_OP_NOOP;
    SyncP gstart = ktime_ && !empty_group ? new_sync(d, s, true) : nullptr;
    const int64_t tpop = now_ns();
    for (Task* t : group) {
      t->state = SFX_STATE_EXECUTING;
      t->stream = s;
      t->t_pop = tpop;
      t->end = gend;
      t->start = gstart;
      record(graphs_[t->gid].get(), SFX_EV_POP, tpop, d * (nstreams_ + nurgent_ + ncoop_) + s, t->tid);
    }
    acts.clear();
    ops.assign(group.size(), OpLaunch());
    std::string err;
    int rc = 0;
    size_t planned = 0;
    while (planned < group.size()) {
      const size_t mark = acts.size();
      rc = plan(d, s, group[planned], acts, ops[planned], err, false);
      if (rc == 0) {
        ++planned;
        continue;
      }
      if (rc != 1) break;
      if (planned > 0) {
        // resources exhausted mid-group: launch what is planned, requeue the rest
        (void)mark;
        if (debug_staging())
          fprintf(stderr, "[sfx] midgroup requeue planned=%zu of %zu first=%llu\n", planned, group.size(),
                  (unsigned long long)group[0]->tid);
        for (size_t k = group.size(); k-- > planned;) {
          Task* t = group[k];
          t->end.reset();
          t->start.reset();
          t->state = SFX_STATE_READY;
          D.queue.push_front(t);
          // give its commutative guards back -- handing them to parked members,
          // who would otherwise wait on a free handle; it re-acquires when popped
          if (t->guards_held) release_commute(t);
        }
        group.resize(planned);
        ops.resize(planned);
        rc = 0;
        break;
      }
      // nothing planned yet: issue the write-backs planned so far, then wait for
      // any completion and re-plan.  The completion count is sampled NOW, before
      // the lock is released for the issue: a completion that lands while the
      // write-backs are issued must still wake this wait (it used to be sampled
      // after re-locking, which could miss the last in-flight task and hang).
      uint64_t total_before = 0;
      for (auto& dv : devs_) total_before += dv->stats.tasks_executed;
      if (debug_staging()) {
        fprintf(stderr, "[sfx] nothing-planned wait group=%zu first=%llu acts=%zu ninflight=%d free=%llu blocks:",
                group.size(), (unsigned long long)group[0]->tid, acts.size(), D.ninflight,
                (unsigned long long)D.free_bytes);
        for (auto& kv : D.blocks)
          fprintf(stderr, " [hid=%llu off=%llu pins=%d valid=%d dirty=%d pf=%d zombie=%d]", (unsigned long long)kv.first,
                  (unsigned long long)kv.second->off, kv.second->pins, kv.second->valid ? 1 : 0,
                  kv.second->dirty ? 1 : 0, kv.second->prefetched ? 1 : 0, kv.second->zombie ? 1 : 0);
        fprintf(stderr, " task accesses:");
        for (auto& a : group[0]->acc) fprintf(stderr, " %llu", (unsigned long long)a.h->hid);
        fprintf(stderr, "\n");
      }
      if (!acts.empty()) {
        lk.unlock();
        std::string e2;
        std::vector<Task*> none;
        std::vector<OpLaunch> noops;
        int r2 = issue(d, s, none, acts, noops, e2);
        lk.lock();
        acts.clear();
        if (r2) {
          rc = SFX_ERR_CUDA;
          err = e2;
          break;
        }
      }

      done_cv_.wait(lk, [&] {
        uint64_t tot = 0;
        for (auto& dv : devs_) tot += dv->stats.tasks_executed;
        return stopping_ || fail_code_ || tot != total_before;
      });
      if (debug_staging()) fprintf(stderr, "[sfx] executor woke (first=%llu)\n", (unsigned long long)group[0]->tid);
      if (stopping_ || fail_code_) {
        rc = -100;
        break;
      }
    }
    if (rc == -100) continue;
    if (rc < 0) {
      poison(rc, err);
      continue;
    }
    {
      // every stream wait first, then the group's start stamp, then copies:
      // waiting earlier is always safe and keeps start >= every predecessor's end
      // -- except waits on this group's own staging copies (copy stream, not yet
      // recorded: they follow their RECORD) and the copy stream's own waits
      std::vector<Action> ordered;
      ordered.reserve(acts.size() + 1);
      const int pfs = pf_stream();
      auto hoist = [&](const Action& a) {
        return a.kind == Action::WAIT && a.stream < 0 &&
               !(a.sync->dev == d && a.sync->stream == pfs && !a.sync->recorded.load(std::memory_order_acquire));
      };
      for (auto& a : acts)
        if (hoist(a)) ordered.push_back(a);
      if (gstart && !ktime_kernel_only_) ordered.push_back(Action{Action::RECORD, gstart});
      for (auto& a : acts)
        if (!hoist(a)) ordered.push_back(a);
      if (gstart && ktime_kernel_only_) ordered.push_back(Action{Action::RECORD, gstart});
      acts.swap(ordered);
    }
    D.ninflight += static_cast<int>(group.size());
    D.stream_inflight[s] += static_cast<int>(group.size());
    D.stream_groups[s] += 1;
    if (stage_window_) {
      gend->staged = group_stage;
      D.stage_inflight += group_stage;
    }
    const int64_t t_plan1 = now_ns();
    D.stats.t_plan_ns += t_plan1 - t_busy0;
    lk.unlock();
    rc = issue(d, s, group, acts, ops, err);
    const int64_t t_issue1 = now_ns();
    D.stats.t_issue_ns += t_issue1 - t_plan1;
    D.stats.groups += 1;
    lk.lock();
    if (rc) {
      poison(rc == SFX_ERR_USER ? SFX_ERR_USER : SFX_ERR_CUDA, err);
      continue;
    }
    const int64_t t_rel0 = now_ns();
    if (!be_->is_sim() && ndev_ == 1)
      // Exclusive commutative guards pass at LAUNCH on one device, like every other
      // dependency: the next member's plan waits on commute_last (this task's end
      // event, set in plan), so members still never overlap on the device, but the
      // next one is issued without a host round trip through the completion thread
      // (the reference holds the guard until the body returns, handles.py:249-270;
      // with several devices the guard stays held to completion: a member placed
      // elsewhere would pull the handle's data while this one may still run)
      for (Task* t : group)
        if (t->guards_held && t->op != SFX_OP_EXTERN && exclusive_guards(t)) release_commute(t);
    if (be_->is_sim()) {
      for (Task* t : group) {
        if (t->op == SFX_OP_EXTERN) {
          extern_handoff(t);  // released by extern_done
          continue;
        }
        complete(t);  // synchronous device: stage_out + task_end before release
        release(t);
      }
    } else {
      for (Task* t : group)
        if (t->op != SFX_OP_EXTERN) release(t);  // extern: released by extern_done
      for (Task* t : group) D.inflight.push_back(t);
      D.comp_cv.notify_one();
    }
    D.stats.t_release_ns += now_ns() - t_rel0;
  }
}

void Runtime::comp_loop(int d) {
  // Completion: a snapshot of the in-flight launch groups is polled OUTSIDE the
  // runtime lock (cudaEventQuery; a blocking sync on the oldest one only when
  // none has finished), their event times are resolved there too, and every
  // finished task is then completed in ONE lock section -- in any order across
  // streams, so a long group on one stream does not hold up the unpinning and
  // guard hand-over of groups that finished on others.
  be_->bind_thread(d);
  Device& D = *devs_[d];
  struct Item {
    Task* t;
    SyncP end, start;
  };
  std::vector<Item> snap;
  std::vector<Task*> keep, fin;
  std::unique_lock<std::mutex> lk(mu_);
  while (true) {
    D.comp_cv.wait(lk, [&] { return stopping_ || !D.inflight.empty(); });
    if (D.inflight.empty()) {
      if (stopping_) return;
      continue;
    }
    snap.clear();
    const size_t K = std::min<size_t>(D.inflight.size(), 512);
    for (size_t i = 0; i < K; ++i) {
      Task* t = D.inflight[i];
      snap.push_back(Item{t, t->end, t->start});
    }
    lk.unlock();
    std::string err;
    int rc = 0;
    // distinct end points in snapshot order (members of a group share one)
    Sync* last = nullptr;
    bool any = false;
    for (size_t i = 0; i < snap.size() && !rc; ++i) {
      Sync* e = snap[i].end.get();
      if (e == last || e->seen_done) continue;
      last = e;
      const int q = be_->event_query(d, e->event, err);
      if (q < 0) rc = q;
      if (q == 1) {
        e->seen_done = true;
        any = true;
      }
    }
    if (!rc && !any && !snap[0].end->seen_done) {  // nothing finished yet: block on the oldest
      rc = be_->event_sync(d, snap[0].end->event, err);
      if (!rc) snap[0].end->seen_done = true;
    }
    if (!rc && ktime_) {
      for (const Item& it : snap) {
        Sync* e = it.end.get();
        if (e->t_resolved || !e->seen_done || !e->timing) continue;
        e->t_ns = be_->event_time_ns(d, e->event);
        e->t_resolved = true;
        if (it.start) {
          it.start->t_ns = be_->event_time_ns(d, it.start->event);
          it.start->t_resolved = true;
        }
      }
    }
    lk.lock();
    const int64_t tc0 = now_ns();
    if (rc) {
      // the context reports an error: fail the engine; the oldest task is retired
      // so that waiters are woken (the engine is poisoned either way)
      poison(rc == SFX_ERR_USER ? SFX_ERR_USER : SFX_ERR_CUDA, err);
      Task* t = D.inflight.front();
      D.inflight.pop_front();
      if (t->op == SFX_OP_EXTERN) {
        extern_handoff(t);
      } else {
        complete(t);
      }
      continue;
    }
    // rebuild the front of the deque: finished tasks leave, the rest keep order
    keep.clear();
    fin.clear();
    for (size_t i = 0; i < snap.size(); ++i) {
      Task* t = D.inflight.front();
      D.inflight.pop_front();
      (snap[i].end->seen_done ? fin : keep).push_back(t);
    }
    for (size_t i = keep.size(); i-- > 0;) D.inflight.push_front(keep[i]);
    for (Task* t : fin) {
      if (t->op == SFX_OP_EXTERN) {
        extern_handoff(t);  // its host copy is current: over to the agent
        continue;
      }
      complete(t);
    }
    D.stats.t_complete_ns += now_ns() - tc0;
  }
}

// ----------------------------------------------------------- waiting/export

int Runtime::pause(bool p) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  paused_ = p;
  if (!p)
    for (auto& d : devs_) d->exec_cv.notify_all();
  return SFX_OK;
}

int Runtime::wait_all(uint32_t gid, double timeout_s) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  auto it = graphs_.find(gid);
  if (it == graphs_.end()) {
    last_error = fmt("unknown graph %u", gid);
    return SFX_ERR_CONFIG;
  }
  Graph* g = it->second.get();
  auto done = [&] { return fail_code_ != 0 || g->completed >= g->inserted; };
  if (timeout_s < 0) {
    done_cv_.wait(lk, done);
  } else {
    done_cv_.wait_for(lk, std::chrono::duration<double>(timeout_s), done);
  }
  if (fail_code_) {
    last_error = fail_msg_;
    return SFX_ERR_ENGINE_FAILED;
  }
  return g->completed >= g->inserted ? SFX_OK : SFX_TIMEOUT;
}

int Runtime::wait_task(uint64_t tid, double timeout_s) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  Task* t = tasks_by_tid_.get(tid);
  if (!t) {
    if (tid && tid <= max_tid_ && retired_tasks_) return SFX_OK;  // retired: it finished
    last_error = "unknown task";
    return SFX_ERR_CONFIG;
  }
  auto done = [&] { return t->state == SFX_STATE_FINISHED || fail_code_ != 0; };
  if (timeout_s < 0)
    done_cv_.wait(lk, done);
  else
    done_cv_.wait_for(lk, std::chrono::duration<double>(timeout_s), done);
  if (t->state == SFX_STATE_FINISHED) return SFX_OK;
  if (fail_code_) {
    last_error = fail_msg_;
    return SFX_ERR_ENGINE_FAILED;
  }
  return SFX_TIMEOUT;
}

int Runtime::task_state(uint64_t tid, int32_t* st) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  Task* found = tasks_by_tid_.get(tid);
  if (!found) {
    if (tid && tid <= max_tid_ && retired_tasks_) {  // retired by a history-free graph: it finished
      *st = SFX_STATE_FINISHED;
      return SFX_OK;
    }
    last_error = "unknown task";
    return SFX_ERR_CONFIG;
  }
  *st = found->state;
  return SFX_OK;
}

int Runtime::stats(int dev, sfx_dev_stats* out) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  if (dev < 0 || dev >= ndev_) {
    last_error = "bad device index";
    return SFX_ERR_CONFIG;
  }
  Device& D = *devs_[dev];
  D.stats.first_start_ns = 0;
  D.stats.last_end_ns = 0;
  if (!D.kintervals.empty()) {
    // union of the timed launch-group intervals (overlapping groups on
    // different streams count once)
    std::sort(D.kintervals.begin(), D.kintervals.end());
    D.stats.first_start_ns = D.kintervals.front().first;
    for (auto& iv : D.kintervals) D.stats.last_end_ns = std::max<int64_t>(D.stats.last_end_ns, iv.second);
    int64_t cs = D.kintervals[0].first, ce = D.kintervals[0].second;
    for (auto& iv : D.kintervals) {
      if (iv.first > ce) {
        D.stats.busy_ns += static_cast<uint64_t>(ce - cs);
        cs = iv.first;
      }
      ce = std::max(ce, iv.second);
    }
    D.stats.busy_ns += static_cast<uint64_t>(ce - cs);
    D.kintervals.clear();
  }
  *out = D.stats;
  if (!be_->is_sim()) out->kernel_launches = be_->kernel_launches();  // process-wide kernel count
  return SFX_OK;
}

int Runtime::resident(int dev, uint64_t* hids, uint64_t cap, uint64_t* n) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  if (dev < 0 || dev >= ndev_) {
    last_error = "bad device index";
    return SFX_ERR_CONFIG;
  }
  uint64_t k = 0;
  for (auto& kv : devs_[dev]->blocks) {
    if (hids && k < cap) hids[k] = kv.first;
    ++k;
  }
  *n = k;
  return SFX_OK;
}

int Runtime::block_state(uint64_t hid, int dev, int32_t* st, int32_t* host_valid) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  Handle* h = nullptr;
  for (auto& hp : handle_store_)
    if (hp->hid == hid) h = hp.get();
  if (!h || dev < 0 || dev >= ndev_) {
    last_error = "unknown handle or device";
    return SFX_ERR_CONFIG;
  }
  Block* b = h->blocks[dev];
  *st = b ? ((b->valid ? 1 : 0) | (b->dirty ? 2 : 0) | 4) : 0;
  *host_valid = h->host_valid ? 1 : 0;
  return SFX_OK;
}

int Runtime::trace(uint32_t gid, sfx_event* buf, uint64_t cap, uint64_t* n) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  auto it = graphs_.find(gid);
  if (it == graphs_.end()) {
    last_error = "unknown graph";
    return SFX_ERR_CONFIG;
  }
  auto& ev = it->second->events;
  std::stable_sort(ev.begin(), ev.end(), [](const sfx_event& a, const sfx_event& b) { return a.t_ns < b.t_ns; });
  *n = ev.size();
  if (buf) memcpy(buf, ev.data(), std::min<uint64_t>(cap, ev.size()) * sizeof(sfx_event));
  return SFX_OK;
}

int Runtime::edges(uint32_t gid, uint64_t* src, uint64_t* dst, uint64_t* hid, uint64_t cap, uint64_t* n) {
  // trace.py:94-102 / 122-127: every member of slot i -> every member of slot i+1
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  auto it = graphs_.find(gid);
  if (it == graphs_.end()) {
    last_error = "unknown graph";
    return SFX_ERR_CONFIG;
  }
  uint64_t k = 0;
  for (Handle* h : it->second->handles) {
    for (size_t i = 0; i + 1 < h->slots.size(); ++i)
      for (Task* a : h->slots[i].tasks)
        for (Task* b : h->slots[i + 1].tasks) {
          if (k < cap) {
            if (src) src[k] = a->tid;
            if (dst) dst[k] = b->tid;
            if (hid) hid[k] = h->hid;
          }
          ++k;
        }
  }
  *n = k;
  return SFX_OK;
}

int Runtime::violations(uint64_t* n) {
  // race detection on device timestamps: every edge must satisfy
  // start(dst) >= end(src) (handles.py:88-107 restated for streams)
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  uint64_t bad = 0;
  for (auto& hp : handle_store_) {
    Handle* h = hp.get();
    for (size_t i = 0; i + 1 < h->slots.size(); ++i)
      for (Task* a : h->slots[i].tasks)
        for (Task* b : h->slots[i + 1].tasks) {
          if (a->state != SFX_STATE_FINISHED || b->state != SFX_STATE_FINISHED) continue;
          if (!a->t_end || !b->t_start) continue;
          // devices on one GPU share one clock: no slack; across GPUs the host-side
          // calibration of each device's base event is good to a few microseconds
          const int64_t slack = be_->same_clock(a->dev, b->dev) ? 0 : 20000;
          if (b->t_start + slack < a->t_end) ++bad;
        }
  }
  *n = bad;
  return SFX_OK;
}

int Runtime::set_option(const std::string& key, int64_t value) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  if (key == "group_max") {
    group_max_ = static_cast<uint32_t>(std::max<int64_t>(1, std::min<int64_t>(value, 1024)));
  } else if (key == "groups_per_stream") {
    groups_per_stream_ = static_cast<uint32_t>(std::max<int64_t>(1, value));
    for (auto& d : devs_) d->exec_cv.notify_all();
  } else if (key == "urgent_priority") {
    urgent_priority_ = value;
  } else if (key == "prefetch") {
    prefetch_ = value != 0 && !be_->is_sim();
  } else if (key == "stage_stream") {
    stage_stream_ = value != 0 && !be_->is_sim();
  } else if (key == "flush_priority") {
    flush_priority_ = static_cast<int32_t>(value);
  } else if (key == "stage_window") {
    stage_window_ = static_cast<uint64_t>(std::max<int64_t>(0, value));
    for (auto& d : devs_) d->wake_exec();
  } else if (key == "prefetch_depth") {
    prefetch_depth_ = static_cast<int>(std::max<int64_t>(0, value));
  } else if (key == "kernel_timing") {
    // launch-group timing events (SFX_FLAG_KTIME); tracing keeps them on
    ktime_ = trace_ || value != 0;
  } else if (key == "deterministic") {
    deterministic_ = value != 0;
  } else if (key == "stream_affinity") {
    stream_affinity_ = value != 0;
  } else if (key == "kernel_only_start") {
    ktime_kernel_only_ = value != 0;
  } else if (key == "window") {
    window_ = static_cast<uint32_t>(std::max<int64_t>(1, value));
    for (auto& d : devs_) d->exec_cv.notify_all();
  } else {
    last_error = "unknown option " + key;
    return SFX_ERR_CONFIG;
  }
  return SFX_OK;
}

int Runtime::graph_option(uint32_t gid, const std::string& key, int64_t value) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  auto it = graphs_.find(gid);
  if (it == graphs_.end()) {
    last_error = fmt("unknown graph %u", gid);
    return SFX_ERR_CONFIG;
  }
  if (key == "history") {
    if (!value && it->second->inserted) {
      last_error = "history can only be switched off before the graph's first task";
      return SFX_ERR_CONFIG;
    }
    it->second->history = value != 0;
    return SFX_OK;
  }
  if (key == "trace") {
    it->second->trace = value != 0;
    return SFX_OK;
  }
  last_error = "unknown graph option " + key;
  return SFX_ERR_CONFIG;
}

int Runtime::live(uint64_t* tasks, uint64_t* slots, uint64_t* retired) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  uint64_t ns = 0;
  for (auto& h : handle_store_) ns += h->slots.size();
  if (tasks) *tasks = live_tasks_;
  if (slots) *slots = ns;
  if (retired) *retired = retired_tasks_;
  return SFX_OK;
}

int Runtime::failure(int* code, char* msg, uint64_t cap) {
  std::unique_lock<std::mutex> lk(mu_);
  drain_locked();
  *code = fail_code_;
  if (msg && cap) {
    strncpy(msg, fail_msg_.c_str(), cap - 1);
    msg[cap - 1] = 0;
  }
  return SFX_OK;
}

}  // namespace sfx
