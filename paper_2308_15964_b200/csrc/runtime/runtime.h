// Native STF runtime: dependency core, locality-aware per-device schedulers,
// per-device tile arenas (LRU + valid/dirty coherency), stream executors with
// CUDA-event release, and completion tracking.
//
// Semantics follow the reference seqflow runtime (paths relative to
// /root/reference/pkg/src/seqflow):
//   slot grouping ........ handles.py:209-236  (Runtime::bind)
//   pending counter ...... task.py:76,105-124  (Task::pending, insertion guard)
//   release / advance .... handles.py:274-343  (Runtime::release)
//   FIFO / priority ...... scheduler.py:66-126 (DevQueue)
//   staging / LRU ........ device.py:197-378   (Runtime::plan_access, evict)
//   coherency ............ device.py:282-326   (dirty_dev / host_valid)
//
// B200-first differences:
//   * a task is released when it is LAUNCHED, not when it finishes: its
//     successors are enqueued behind a cudaStreamWaitEvent on its end event,
//     so the host never sits on the critical path; completion is tracked by
//     a per-device thread that only unpins blocks and does accounting;
//   * cross-device reads pull the freshest copy peer-to-peer (NVLink) from
//     the dirty owner instead of bouncing through the host;
//   * commutative members are serialized per handle by chaining on the
//     previous member's end event (any order, never concurrent).
#pragma once
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "sfx.h"

namespace sfx {

enum Cat : uint8_t { CAT_R = 0, CAT_A = 1, CAT_C = 2, CAT_X = 3 };

inline Cat category_of(uint32_t mode) {
  switch (mode) {
    case SFX_READ: return CAT_R;
    case SFX_ATOMIC_WRITE: return CAT_A;
    case SFX_COMMUTATIVE_WRITE: return CAT_C;
    default: return CAT_X;  // WRITE and MAYBE_WRITE are exclusive (access.py:41-47)
  }
}
inline bool mode_writes(uint32_t m) { return m != SFX_READ; }
// ops whose writes to commutative operands are device-atomic accumulations:
// concurrent members of a commutative group give one of the results a serial
// order would (up to FP rounding), so their guard is taken in shared mode
inline bool accumulates_atomically(uint32_t op) {
  return op == SFX_OP_P2P_PAIR || op == SFX_OP_P2P_SELF || op == SFX_OP_ADD_I64;
}

class Backend;

// A point recorded on one device stream (a CUDA event), shared by everything
// that must wait for it.  `recorded` flips once the executor that planned it
// has issued the record, so a waiter planned meanwhile can spin briefly.
struct Sync {
  Backend* be = nullptr;
  int dev = -1, stream = -1;
  void* event = nullptr;
  bool timing = false;
  std::atomic<bool> recorded{false};
  bool complete = false;       // guarded by the runtime mutex
  bool group_counted = false;  // launch group already retired from its stream
  uint64_t staged = 0;         // launch group: bytes it staged from the host (stage window)
  bool group_timed = false;    // launch group duration already accumulated (KTIME)
  int64_t t_ns = 0;            // host-clock time of the event, resolved by the completion
  bool t_resolved = false;     // thread OUTSIDE the runtime mutex (only it touches these)
  bool seen_done = false;      // completion thread: this point was observed complete
  ~Sync();
};
using SyncP = std::shared_ptr<Sync>;

struct Task;
struct Handle;

struct Slot {
  Cat cat;
  std::vector<Task*> tasks;
  uint32_t done = 0;      // members released (at launch)
  uint32_t finished = 0;  // members completed (retirement: history-free graphs)
};

struct Graph;

struct Block {
  Handle* h = nullptr;
  int dev = -1;
  uint64_t off = 0, size = 0;
  uint64_t stamp = 0;
  int pins = 0;
  bool valid = false, dirty = false, zombie = false;
  bool prefetched = false;  // holds one pin for a not-yet-launched reader (prefetch)
  SyncP ready;  // contents valid once this completes (null: valid now)
};

struct Handle {
  uint64_t hid = 0;
  uint32_t gid = 0;
  void* host = nullptr;
  uint64_t bytes = 0;
  int64_t rows = 0, cols = 0, ld = 0;
  int32_t dtype = 0;
  // slots by ABSOLUTE index (Access::slot, active): slots.front() is slot_base;
  // a history-free graph pops slots that are passed and whose members all finished
  std::deque<Slot> slots;
  uint32_t slot_base = 0;
  uint32_t slot_end() const { return slot_base + static_cast<uint32_t>(slots.size()); }
  Slot& slot(uint32_t abs) { return slots[abs - slot_base]; }
  uint32_t active = 0;
  Graph* graph = nullptr;
  std::vector<Block*> blocks;  // per device
  int dirty_dev = -1;          // at most one dirty copy
  bool host_valid = true;
  SyncP host_ready;     // host buffer is current once this completes
  SyncP commute_last;   // end of the last launched commutative member
  // commutative exclusivity guard (handles.py:249-270): held from launch until
  // the owner COMPLETES; tasks that fail to acquire park on the handle instead
  // of being re-offered (no quadratic re-offer scan, handles.py:317-328)
  Task* commute_owner = nullptr;
  std::deque<Task*> commute_waiters;
  // shared mode (ops that accumulate with device atomics, accumulates_atomically):
  // members run concurrently on ONE device; exclusive members wait for them all
  int shared_users = 0;
  int shared_dev = -1;
  int group_dev = -1;   // device of the active atomic/commutative group
  int home = -1;        // owner hint (2-D block-cyclic distribution)
  bool superseded = false;  // its host memory was registered by another graph (see reg)
};

struct Access {
  Handle* h;
  uint32_t mode;
  uint32_t slot;
};

struct Task {
  uint64_t tid = 0;
  uint32_t gid = 0, op = 0;
  int32_t prio = 0, hint = -1;
  double fp[4] = {0, 0, 0, 0};
  int64_t ip[4] = {0, 0, 0, 0};
  std::vector<Access> acc;
  int32_t pending = 1;  // insertion guard (task.py:76)
  int state = SFX_STATE_INSERTED;
  bool released = false;
  uint64_t seq = 0;  // scheduler push sequence
  int dev = -1, stream = -1;
  std::vector<SyncP> waits;       // predecessors' end points
  SyncP start, end;
  std::vector<Block*> pinned;     // unpinned at completion
  std::vector<SyncP> copy_syncs;  // copies issued on this task's stream
  int64_t t_push = 0, t_pop = 0, t_start = 0, t_end = 0;
  // guarded handles sorted by hid (graph.py:150-157): its commutative handles, and on
  // a multi-device runtime its atomic ones; commute_sh[k]: guard k in shared mode
  // (members run concurrently on ONE device: an op that accumulates with device
  // atomics, or any atomic_write member)
  std::vector<Handle*> commute;
  std::vector<uint8_t> commute_sh;
  bool guards_held = false;      // its commutative guards are acquired (idempotent acquire)
  bool detached = false;         // SFX_OP_EXTERN handed to the host agent: stream slots freed
  int status_slot = -1;          // device-written status word (DPOTRF info), read at completion
  uint32_t slot_refs = 0;        // slots of it not yet retired (freed back to the pool at 0)
};

struct Operand {
  void* dptr = nullptr;
  uint64_t bytes = 0;
  int64_t rows = 0, cols = 0, ld = 0;
  int32_t dtype = 0;
  uint32_t mode = 0;  // the task's access mode for this operand (user ops' views)
};

struct OpLaunch {
  uint32_t op = 0;
  int n = 0;
  int status_slot = -1;  // Backend::status_alloc slot the kernel reports into (DPOTRF info)
  bool deterministic = false;  // Runtime deterministic mode: order-independent launches
  Operand o[8];
  double fp[4];
  int64_t ip[4];
};

// User ops (sfx_register_op): process-wide table of host-side launchers, written
// once per code and read without a lock afterwards.
struct UserOp {
  char name[64];
  sfx_user_launch_fn fn;
  void* user;
};
const UserOp* user_op(uint32_t op);  // nullptr unless op is a registered user op
int register_user_op(const char* name, sfx_user_launch_fn fn, void* user, uint32_t* op, std::string& err);
// calls the launcher with the staged operands as views; SFX_ERR_USER on failure
int run_user_op(const UserOp& u, const OpLaunch& op, int dev, void* stream, std::string& err);

// Task lookup by tid (sfx_wait_task, sfx_task_state, extern_done, duplicate
// check).  Tids are process-global increasing counters, so a paged direct table
// (64 Ki tids per page, freed when its last task retires) replaces a hash map:
// the map's rehash of ~10^6 entries stalled insertion for ~100 ms once it grew
// past a bucket-count threshold (a C2 step after a 20-step burst).
class TidMap {
 public:
  Task* get(uint64_t tid) const {
    auto it = pages_.find(tid >> kBits);
    return it == pages_.end() ? nullptr : it->second.slot[tid & kMask];
  }
  size_t count(uint64_t tid) const { return get(tid) ? 1 : 0; }
  void put(uint64_t tid, Task* t) {
    Page& p = pages_[tid >> kBits];
    if (!p.slot) p.slot.reset(new Task*[size_t(1) << kBits]());
    if (!p.slot[tid & kMask]) p.live += 1;
    p.slot[tid & kMask] = t;
  }
  void erase(uint64_t tid) {
    auto it = pages_.find(tid >> kBits);
    if (it == pages_.end() || !it->second.slot[tid & kMask]) return;
    it->second.slot[tid & kMask] = nullptr;
    if (--it->second.live == 0) pages_.erase(it);
  }

 private:
  static constexpr int kBits = 16;
  static constexpr uint64_t kMask = (uint64_t(1) << kBits) - 1;
  struct Page {
    std::unique_ptr<Task*[]> slot;
    size_t live = 0;
  };
  std::unordered_map<uint64_t, Page> pages_;
};

// One step of a planned task, issued outside the runtime lock.
struct Action {
  enum Kind { WAIT, H2D, D2H, P2P, RECORD } kind;
  SyncP sync;
  uint64_t dst_off = 0, src_off = 0, n = 0;
  void* host = nullptr;
  int src_dev = -1;
  int stream = -1;  // >= 0: issued on this stream instead of the group's (host staging stream)
};

// Device/stream abstraction: CUDA (B200) or host-memory simulation (tests).
class Backend {
 public:
  virtual ~Backend() {}
  virtual bool is_sim() const = 0;
  // nstreams normal-priority streams, then nurgent highest-priority streams, then
  // ncoop highest-priority streams reserved for cooperative (grid-barrier) kernels
  virtual int init_device(int d, int ordinal, int nstreams, int nurgent, int ncoop, int nprefetch,
                          uint64_t arena_bytes, std::string& err) = 0;
  virtual void bind_thread(int d) = 0;
  // timestamps of devices a and b come from one clock (same physical GPU)
  virtual bool same_clock(int a, int b) const { return a == b; }
  virtual uint64_t arena_capacity(int d) = 0;
  virtual void* arena_ptr(int d, uint64_t off) = 0;
  virtual void* event_create(int d, bool timing) = 0;
  virtual void event_release(int d, void* ev) = 0;
  virtual int event_record(int d, int stream, void* ev, std::string& err) = 0;
  virtual int stream_wait(int d, int stream, void* ev, std::string& err) = 0;
  virtual int event_sync(int d, void* ev, std::string& err) = 0;
  // true once the recorded work before ev has executed (sim: always)
  virtual bool event_done(int d, void* ev) = 0;
  // 1 = done, 0 = not yet, < 0 = error (err set): the completion thread's poll
  virtual int event_query(int d, void* ev, std::string& err) { return event_done(d, ev) ? 1 : 0; }
  // CLOCK_MONOTONIC ns of a completed timing event
  virtual int64_t event_time_ns(int d, void* ev) = 0;
  virtual int copy_h2d(int d, int stream, uint64_t dst_off, const void* src, uint64_t n, std::string& err) = 0;
  virtual int copy_d2h(int d, int stream, void* dst, uint64_t src_off, uint64_t n, std::string& err) = 0;
  virtual int copy_p2p(int d, int stream, uint64_t dst_off, int src_dev, uint64_t src_off, uint64_t n,
                       std::string& err) = 0;
  virtual int launch(int d, int stream, const OpLaunch& op, std::string& err) = 0;
  // several independent ready tasks on one stream (grouped kernels where available)
  virtual int launch_group(int d, int stream, const std::vector<OpLaunch>& ops, std::string& err) {
    for (const OpLaunch& op : ops) {
      int rc = launch(d, stream, op, err);
      if (rc) return rc;
    }
    return 0;
  }
  virtual bool supports(uint32_t op) const = 0;
  // status words written by kernels (DPOTRF info: 0 = success, else the 1-based
  // order of the first non-positive leading minor); host-visible once the
  // launching task's end event completed.  -1: none available (sim)
  virtual int status_alloc(int) { return -1; }
  // read the word, reset it to 0 and return the slot to the pool
  virtual int status_take(int, int) { return 0; }
  // kernels launched so far by this process's ops (0 for the simulator)
  virtual uint64_t kernel_launches() const { return 0; }
  virtual void shutdown() = 0;
};

Backend* make_sim_backend(int ndev);
Backend* make_cuda_backend(int ndev, const int* ordinals, bool trace);
int64_t now_ns();

struct Graph {
  uint32_t gid = 0;
  uint64_t inserted = 0, completed = 0;
  // history (default, the reference's behaviour): every task and slot is kept for
  // the dot export / edges.  Without it finished tasks and passed slots are
  // retired (bounded runtime memory for long-running graphs, handles.py:114-189)
  bool history = true;
  bool trace = true;  // TaskGraph(trace=...): record events (when the runtime traces)
  std::vector<Handle*> handles;
  std::vector<sfx_event> events;
};

struct DevQueue {
  // FIFO (scheduler.py:66-94) or max-priority with FIFO ties (scheduler.py:97-126)
  bool prio = false;
  std::deque<Task*> fifo;
  std::vector<Task*> heap;
  size_t size() const { return prio ? heap.size() : fifo.size(); }
  void push(Task* t);
  void push_front(Task* t);
  Task* pop();
  Task* peek() const;
};

struct Device {
  int index = 0;
  uint64_t capacity = 0, free_bytes = 0;
  std::map<uint64_t, uint64_t> free_list;      // offset -> size, first fit
  // arena ranges whose evicted contents are still being written back (D2H on the
  // evicting task's stream): a new block allocated over one must wait for it
  struct PendingWriteBack {
    uint64_t off, size;
    SyncP done;
  };
  std::vector<PendingWriteBack> pending_wb;
  std::unordered_map<uint64_t, Block*> blocks;  // hid -> live block
  uint64_t clock = 0;
  DevQueue queue;
  std::deque<Task*> inflight;
  std::vector<int> stream_inflight;  // tasks in flight per stream
  std::vector<int> stream_groups;    // launch groups in flight per stream
  int ninflight = 0;
  std::condition_variable exec_cv, comp_cv;
  // the executor sleeps on exec_cv: per-task wake-ups (push, completion) signal it
  // only while it sleeps and only once per sleep (no futex storm from a burst of
  // pushes, and none at all while it is busy); guarded by the runtime mutex
  bool exec_sleeping = false;
  void wake_exec() {
    if (exec_sleeping) {
      exec_sleeping = false;
      exec_cv.notify_one();
    }
  }
  std::thread exec_thread, comp_thread;
  sfx_dev_stats stats{};
  std::vector<std::pair<int64_t, int64_t>> kintervals;  // KTIME group [start, end] not yet folded into busy_ns
  bool prefetch_pending = false;  // ready queue changed since the last prefetch pass
  uint64_t stage_inflight = 0;    // host bytes staged by launch groups still in flight
};

class Runtime {
 public:
  Runtime(Backend* be, int ndev, int nstreams, uint32_t sched, uint32_t flags, uint32_t window, uint64_t align);
  ~Runtime();
  int init(const uint64_t* arena_bytes, std::string& err);

  int graph_create(uint32_t* gid);
  int reg(uint32_t gid, uint64_t hid, void* host, uint64_t bytes, int64_t rows, int64_t cols, int64_t ld,
          int32_t dtype);
  int set_home(uint64_t hid, int dev);
  int unreg(uint64_t hid);
  int submit(uint32_t n, const sfx_task_desc* tasks, const sfx_access* acc);
  // bind + push (check: validate each first); the caller holds mu_
  int submit_bound(uint32_t n, const sfx_task_desc* tasks, const sfx_access* acc, bool check);
  // binds the submissions queued by submit() (ring mode); the caller holds mu_
  void drain_locked();
  int flush(uint32_t gid, uint64_t tid, uint64_t hid, int write_mode);
  int pause(bool p);
  int wait_all(uint32_t gid, double timeout_s);
  int wait_task(uint64_t tid, double timeout_s);
  int task_state(uint64_t tid, int32_t* st);
  int stats(int dev, sfx_dev_stats* out);
  int extern_poll(uint64_t* tids, uint64_t cap, uint64_t* n, double timeout_s);
  int extern_done(uint64_t tid, int status, const char* msg);
  int fail(const std::string& msg);
  int resident(int dev, uint64_t* hids, uint64_t cap, uint64_t* n);
  int block_state(uint64_t hid, int dev, int32_t* st, int32_t* host_valid);
  int trace(uint32_t gid, sfx_event* buf, uint64_t cap, uint64_t* n);
  int edges(uint32_t gid, uint64_t* src, uint64_t* dst, uint64_t* hid, uint64_t cap, uint64_t* n);
  int violations(uint64_t* n);
  int failure(int* code, char* msg, uint64_t cap);
  int set_option(const std::string& key, int64_t value);
  int graph_option(uint32_t gid, const std::string& key, int64_t value);
  int live(uint64_t* tasks, uint64_t* slots, uint64_t* retired);

  std::string last_error;

 private:
  int validate(const sfx_task_desc& d, const sfx_access* acc, std::string& err);
  int retire_blocks(Handle* h);  // write dirty copies home (synchronously), drop every block
  void bind(Task* t, Handle* h, uint32_t mode);
  void push_ready(Task* t, int wid);
  int place(Task* t);
  void release(Task* t);
  void advance(Handle* h);
  int plan(int d, int s, Task* t, std::vector<Action>& acts, OpLaunch& op, std::string& err, bool record_start);
  bool groupable(const Task* t) const;
  bool same_signature(const Task* a, const Task* b) const;
  bool commute_conflict(const std::vector<Task*>& group, const Task* t) const;
  bool acquire_commute(Task* t);
  void release_commute(Task* t);
  int ensure_block(int d, int s, Handle* h, std::vector<Action>& acts, std::vector<Block*>& tmp_pins, Block** out,
                   std::string& err);
  void wait_pending_wb(int d, int s, uint64_t off, uint64_t size, std::vector<Action>& acts);
  int evict_one(int d, int s, std::vector<Action>& acts, std::string& err);
  void drop_block(Block* b, bool write_back, std::vector<Action>* acts, int s);
  void free_space(int d, uint64_t off, uint64_t size);
  bool alloc_space(int d, uint64_t size, uint64_t* off);
  SyncP new_sync(int d, int s, bool timing);
  int issue(int d, int s, const std::vector<Task*>& group, std::vector<Action>& acts, std::vector<OpLaunch>& ops,
            std::string& err);
  void complete(Task* t);
  void poison(int code, const std::string& msg);
  void record(Graph* g, int kind, int64_t t, int wid, uint64_t tid, int64_t extra = 0);
  void exec_loop(int d);
  void comp_loop(int d);

  Backend* be_;
  int ndev_, nstreams_;
  uint32_t sched_, flags_, window_;
  uint32_t group_max_ = 32;
  uint32_t groups_per_stream_ = 2;  // launches queued ahead on each stream
  // tasks with priority >= urgent_priority_ go to the high-priority CUDA
  // streams (indices nstreams_ .. nstreams_+nurgent_-1): the block scheduler
  // then starts their CTAs first whenever an SM frees up (critical path)
  int nurgent_ = 0;
  int64_t urgent_priority_ = 1000000;
  // cooperative POTRF/TRSM kernels run only on these (at most ncoop_ of them
  // co-resident, so their grid barriers can never starve each other)
  int ncoop_ = 2;
  bool stream_affinity_ = true;  // successors join their in-flight predecessor's stream
  bool ktime_kernel_only_ = false;  // the group's start stamp after its copies (timeline diagnostics)
  // deterministic mode: no order-dependent FP64 accumulation anywhere -- ops that
  // normally accumulate with device atomics run one-sided kernels under
  // exclusive guards, DGEMMs never split K (OpLaunch::deterministic); with one
  // stream and FIFO order repeated runs are bitwise identical
  bool deterministic_ = false;
  bool shared_accum(uint32_t op) const { return !deterministic_ && accumulates_atomically(op); }
  bool is_coop(const Task* t) const;
  // Prefetch: while every stream is busy, the executor stages host-resident
  // operands of tasks waiting in its queue on a dedicated copy stream, so PCIe
  // transfers overlap compute (never evicts; keeps capacity/8 free).
  bool prefetch_ = true;
  // host -> device staging of task operands on the device's copy stream (one
  // FIFO in dispatch = priority order) instead of each group's own stream
  bool stage_stream_ = false;
  // > 0: a launch group that has to stage operands from the host waits while the
  // groups in flight already stage this many bytes (keeps the copy FIFO short, so
  // the next priority level's operands are not queued behind a whole wave's)
  uint64_t stage_window_ = 0;
  // priority of flush tasks (the reference's flushes are plain tasks, priority 0);
  // a high value returns finished tiles while lower-priority work still runs
  int32_t flush_priority_ = 0;
  int prefetch_depth_ = 64;
  int pf_stream() const { return nstreams_ + nurgent_ + ncoop_; }
  int plan_prefetch(int d, std::vector<Action>& acts);
  uint64_t align_;
  bool trace_;
  bool ktime_;  // trace_ || SFX_FLAG_KTIME: every launch group gets a timing start event
  std::mutex mu_;
  // Submission ring (SFX_SUBMIT_RING=0: off).  submit() validates on the calling
  // thread (the maps it reads are only changed by API calls of that thread) and
  // queues the descriptors under ring_mu_; whoever holds mu_ next -- an executor
  // at the top of its loop, any API call, or the inserter itself when mu_ is free
  // -- binds them in submission order.  The inserter never waits for mu_ while an
  // executor or a completion thread holds it.  An executor announces its sleep in
  // sleepers_ before the last look at ring_pending_; an inserter that finds a
  // sleeper after queueing drains itself (seq_cst both ways: no lost wake-up).
  bool ring_mode_ = true;
  std::mutex ring_mu_;
  std::vector<sfx_task_desc> ring_descs_, ring_descs_spare_;
  std::vector<sfx_access> ring_acc_, ring_acc_spare_;
  std::atomic<bool> ring_pending_{false};
  std::atomic<int> sleepers_{0};
  std::condition_variable done_cv_;
  std::condition_variable extern_cv_;
  std::deque<Task*> extern_ready_;  // SFX_OP_EXTERN tasks whose host buffers are current
  void extern_handoff(Task* t);
  std::vector<std::unique_ptr<Device>> devs_;
  std::unordered_map<uint64_t, Handle*> handles_;
  // live handles by host start address (cross-graph aliasing check in reg)
  std::multimap<uintptr_t, Handle*> host_ranges_;
  uint64_t max_handle_bytes_ = 0;
  std::vector<std::unique_ptr<Handle>> handle_store_;
  std::unordered_map<uint32_t, std::unique_ptr<Graph>> graphs_;
  TidMap tasks_by_tid_;
  std::vector<std::unique_ptr<Task>> task_store_;  // every Task object ever allocated
  std::vector<Task*> task_free_;                   // retired, reusable
  std::vector<Handle*> retire_pending_;            // handles whose active slot moved (history-free)
  uint64_t max_tid_ = 0, live_tasks_ = 0, retired_tasks_ = 0;
  Task* new_task();
  void free_task(Task* t);
  void flush_retire();
  uint32_t next_gid_ = 1;
  uint64_t push_seq_ = 0;
  bool paused_ = false, stopping_ = false;
  int fail_code_ = 0;
  std::string fail_msg_;
  bool started_ = false;
};

}  // namespace sfx
