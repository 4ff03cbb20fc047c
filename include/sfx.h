/*
 * sfx.h -- C ABI of the B200-native execution path for the Specx/seqflow
 * sequential-task-flow runtime (reference: /root/reference/pkg/src/seqflow).
 *
 * Plain pointers, sizes and integers only; no torch or CUDA types.  Every
 * entry point returns an int status (SFX_OK = 0, negative = error) and the
 * message of the last error on this runtime is available from
 * sfx_last_error().  Calls come from ONE inserter thread per runtime
 * (reference graph.py:85-90); executors, event-completion threads and
 * copies are internal.
 *
 * Reference interface each entry point replaces (file:line relative to
 * pkg/src/seqflow/):
 *   sfx_create / sfx_destroy ...... create_engine engine.py:280, ComputeEngine
 *                                   __init__ engine.py:180-198, stop() 247-258,
 *                                   WorkerTeam.of_host_and_device_workers 58-68
 *   sfx_graph_create .............. TaskGraph.__init__ graph.py:34 +
 *                                   compute_on graph.py:57-64
 *   sfx_register / sfx_unregister . HandleRegistry.ensure/unregister
 *                                   handles.py:159-182 (+ the movable protocol
 *                                   device.py:136-194: a host pointer and a 2-D
 *                                   descriptor replace move_to/from_device)
 *   sfx_submit .................... TaskGraph.task / _insert_raw graph.py:77-166
 *                                   (+ append_access handles.py:209-236,
 *                                   dispatch_ready graph.py:176-182)
 *   sfx_wait_all .................. TaskGraph.wait_all graph.py:199-217
 *   sfx_wait_task ................. TaskViewer.wait task.py:233-239
 *   sfx_flush ..................... TaskGraph.flush_to_host graph.py:258-260
 *   sfx_stats ..................... Mover meters device.py:22-46
 *   sfx_trace ..................... TraceRecorder.export_events trace.py:78-84
 *   sfx_edges ..................... successor_edges / render_dot trace.py:94-135
 *   sfx_pause / sfx_resume ........ the gate task of the reference's gated
 *                                   insertion protocol (tests/conftest.py:184-203)
 */
#ifndef SFX_H
#define SFX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFX_ABI_VERSION 1

/* ---- status codes (map 1:1 onto the reference exception classes) ---- */
#define SFX_OK 0
#define SFX_TIMEOUT 1              /* wait_all: timeout expired (returns False)     */
#define SFX_ERR_CONFIG (-2)        /* ConfigurationError (errors.py:12-13)          */
#define SFX_ERR_STAGING (-3)       /* StagingError (errors.py:36-37)                */
#define SFX_ERR_ENGINE_FAILED (-4) /* EngineFailedError (errors.py:32-33); cause via
                                      sfx_failure()                                 */
#define SFX_ERR_CUDA (-5)          /* CUDA runtime error (cause of an engine failure) */
#define SFX_ERR_INTERNAL (-6)      /* InternalConsistencyError (errors.py:20-21)    */
#define SFX_ERR_DUPLICATE (-7)     /* DuplicateAccessError (errors.py:16-17)        */
#define SFX_ERR_REGISTRATION (-8)  /* RegistrationError (errors.py:8-9)             */
#define SFX_ERR_UNSUPPORTED (-9)   /* op needs a CUDA device (sim backend)          */
#define SFX_ERR_NUMERIC (-10)      /* a tile body reported a numerical failure (DPOTRF:
                                      non-positive pivot, LAPACK info > 0); the cause
                                      of an engine failure, like the LinAlgError the
                                      oracle's np.linalg.cholesky raises              */
#define SFX_ERR_USER (-11)        /* a user op's launcher returned non-zero (the cause of
                                      an engine failure, like a failing device= callable
                                      in the reference, engine.py:154-157)          */

/* ---- access modes (access.py:16-21) ---- */
#define SFX_READ 0
#define SFX_WRITE 1
#define SFX_ATOMIC_WRITE 2
#define SFX_COMMUTATIVE_WRITE 3
#define SFX_MAYBE_WRITE 4

/* ---- runtime flags ---- */
#define SFX_FLAG_SIM 1u    /* host-memory simulated devices: bookkeeping tests only;
                              tile ops are refused with SFX_ERR_UNSUPPORTED       */
#define SFX_FLAG_TRACE 2u  /* record Push/Pop/Start/End (CUDA-event timestamps)     */
#define SFX_FLAG_PAUSED 4u /* start with executors held (gated insertion)           */
#define SFX_FLAG_KTIME 8u  /* time every launch group on its stream (CUDA events):
                              sfx_dev_stats.timed_* (bench roofline)              */

/* ---- schedulers (scheduler.py:66-126) ---- */
#define SFX_SCHED_FIFO 0
#define SFX_SCHED_PRIO 1

/* ---- dtypes ---- */
#define SFX_DTYPE_BYTES 0
#define SFX_DTYPE_F64 1
#define SFX_DTYPE_I64 2

/* ---- ops (operands are the task's accesses in declaration order) ---- */
#define SFX_OP_NOOP 0          /* any accesses; no data movement beyond staging     */
#define SFX_OP_SPIN 1          /* busy-wait iparam[0] ns on the device (overhead bench) */
#define SFX_OP_CELL 2          /* int64 cell arithmetic of the reference random programs
                                  (tests/conftest.py:87-124): iparam = {kind, a, b}   */
#define SFX_OP_BYTES_ADD 3     /* bytes[off:off+len] += delta (mod 256): iparam={off,len,delta} */
#define SFX_OP_FLUSH 4         /* runtime-internal host flush (write or read mode)    */
#define SFX_OP_EXTERN 6        /* one access; executed OUTSIDE the runtime by a host agent
                                  (inter-process send/recv/broadcast, reference
                                  comms.py:303-483): when ready, its host buffer is made
                                  current (read: dirty device copy fetched home; write:
                                  device copies dropped), then the task is handed out by
                                  sfx_extern_poll and finished by sfx_extern_done, which
                                  releases its successors                              */
#define SFX_OP_FAULT 7         /* failure injection for the engine-failure tests: iparam[0] = 0
                                  an invalid launch configuration (the launch itself fails,
                                  non-sticky), 1 a device-side trap (sticky: the CUDA context
                                  is lost; run it in a throw-away process)             */
#define SFX_OP_ADD_I64 5       /* every operand (int64 cells): += iparam[0] with device
                                  atomics.  Like P2P_PAIR/P2P_SELF it accumulates
                                  atomically, so its commutative members of one group run
                                  concurrently on one device (shared guard)            */
#define SFX_OP_DGEMM 10        /* C = beta*C + alpha*A*op(B); fparam={alpha,beta}, iparam[0]=trans_b */
#define SFX_OP_DSYRK 11        /* C = beta*C + alpha*A*A^T, lower; fparam={alpha,beta} */
#define SFX_OP_DTRSM 12        /* B = B * L^-T  (right, lower, transposed, non-unit)   */
#define SFX_OP_DPOTRF 13       /* A = L*L^T in place, lower                            */
#define SFX_OP_P2P_PAIR 20     /* particles: P_i, P_j (read), F_i, F_j (commutative)   */
#define SFX_OP_P2P_SELF 21     /* particles: P_i (read), F_i (commutative)             */
#define SFX_OP_FILL_UNIFORM 30 /* A = splitmix64 uniform[0,1): iparam={seed,row0,col0,ncols_total} */
#define SFX_OP_FILL_SPD 31     /* A = (R+R^T)/2 + n*I tile: iparam={seed,row0,col0,n}    */
#define SFX_OP_FILL_PARTICLES 32 /* P (4 x n SoA x,y,z,q): iparam={seed,first_particle}  */
#define SFX_OP_ZERO 33         /* A = 0                                                  */
#define SFX_OP_DACC 34         /* A += B1 + ... + Bk (FP64, same rows x cols, k = 1..7):
                                  the reduction of per-GPU partial accumulators        */
#define SFX_OP_USER_BASE 256   /* user ops registered with sfx_register_op get the codes
                                  SFX_OP_USER_BASE .. SFX_OP_USER_BASE + SFX_OP_USER_MAX - 1 */
#define SFX_OP_USER_MAX 64

/* ---- trace event kinds (trace.py:14-21) ---- */
#define SFX_EV_PUSH 0
#define SFX_EV_POP 1
#define SFX_EV_START 2
#define SFX_EV_END 3
#define SFX_EV_STAGE_BEGIN 4
#define SFX_EV_STAGE_END 5

/* ---- task states (task.py:11-16) ---- */
#define SFX_STATE_INSERTED 0
#define SFX_STATE_READY 1
#define SFX_STATE_EXECUTING 2
#define SFX_STATE_FINISHED 3

typedef struct sfx_runtime sfx_runtime;

typedef struct sfx_task_desc {
  uint64_t tid;       /* caller-assigned, process-global (task.py:63-69)         */
  uint32_t graph;     /* from sfx_graph_create                                    */
  uint32_t op;        /* SFX_OP_*                                                 */
  int32_t priority;   /* PriorityScheduler key (-priority, seq) scheduler.py:111  */
  int32_t device;     /* placement hint, -1 = locality-aware scheduler decides    */
  uint32_t n_access;  /* this task's accesses, consecutive in the access array    */
  uint32_t flags;     /* reserved, 0                                               */
  double fparam[4];
  int64_t iparam[4];
} sfx_task_desc;

typedef struct sfx_access {
  uint64_t hid;  /* registered handle id */
  uint32_t mode; /* SFX_READ ...          */
  uint32_t reserved;
} sfx_access;

typedef struct sfx_dev_stats {
  /* Mover meters (device.py:26-30) */
  uint64_t bytes_to_device, copies_to_device;     /* host -> device */
  uint64_t bytes_from_device, copies_from_device; /* device -> host */
  uint64_t bytes_p2p_in, copies_p2p_in;           /* peer -> this device (NVLink) */
  /* tile cache */
  uint64_t hits, misses, evictions, writebacks;
  uint64_t blocks, bytes_in_use, capacity;
  /* executor; kernel_launches = CUDA kernels launched by this process's ops
   * (sim: ops executed) */
  uint64_t tasks_executed, kernel_launches, stream_waits;
  /* host-side time of the executor (ns): planning under the lock, issuing
   * stream work outside it, releasing successors; completion-thread time;
   * number of launch groups */
  uint64_t t_plan_ns, t_issue_ns, t_release_ns, t_complete_ns, groups;
  uint64_t prefetches; /* host->device copies staged ahead of the reading task */
  /* SFX_FLAG_KTIME (or TRACE): launch groups timed start->end with CUDA events
   * recorded on the launching stream (after its stream waits), the tasks they
   * carried, the summed group durations and the union of the group intervals
   * (device time with at least one timed group running; folded in when
   * sfx_stats is called) */
  uint64_t timed_groups, timed_tasks, timed_ns, busy_ns;
  /* earliest group start / latest group end (CLOCK_MONOTONIC ns) among the
   * intervals folded in by this sfx_stats call (0 if none) */
  int64_t first_start_ns, last_end_ns;
} sfx_dev_stats;

typedef struct sfx_event {
  int64_t t_ns;   /* CLOCK_MONOTONIC ns (same clock as Python perf_counter_ns) */
  uint64_t tid;
  int32_t kind;   /* SFX_EV_* */
  int32_t worker; /* device * streams_per_dev + stream; -1 inserter            */
  int64_t extra;  /* hid for stage events                                       */
} sfx_event;

int sfx_abi_version(void);
/* number of CUDA devices visible (0 without a driver/GPU) */
int sfx_device_count(int* n);

/* ndev devices (ordinals[i]; NULL = 0..ndev-1), streams_per_dev streams each
 * (WorkerTeam workers_per_device), arena_bytes[i] per device (NULL or 0 =
 * default: free HBM minus a reserve on CUDA, 16 MiB in sim).  window = max
 * in-flight tasks per device (0 = 4 * streams_per_dev). */
int sfx_create(int ndev, const int* ordinals, int streams_per_dev, const uint64_t* arena_bytes,
               uint32_t sched, uint32_t flags, uint32_t window, sfx_runtime** out);
int sfx_destroy(sfx_runtime* rt);
const char* sfx_last_error(sfx_runtime* rt);
/* first failure that poisoned the engine: its status code and message */
int sfx_failure(sfx_runtime* rt, int* code, char* msg, uint64_t cap);

int sfx_graph_create(sfx_runtime* rt, uint32_t* gid);
/* per-graph options: "trace" (default 1: record Push/Pop/Start/End when the
 * runtime traces; TaskGraph(trace=False) switches it off), "history" (default 1: every task and slot is kept for the
 * dot export, as in the reference; 0, before the first task: finished tasks and
 * passed slots are retired -- bounded memory for long-running graphs -- and
 * sfx_edges only reports slots still live) */
int sfx_graph_option(sfx_runtime* rt, uint32_t gid, const char* key, int64_t value);
/* live Task objects, live slots (all handles) and tasks retired so far */
int sfx_live(sfx_runtime* rt, uint64_t* tasks, uint64_t* slots, uint64_t* retired);
int sfx_register(sfx_runtime* rt, uint32_t gid, uint64_t hid, void* host, uint64_t bytes, int64_t rows,
                 int64_t cols, int64_t ld, int32_t dtype);
/* owner hint for the locality-aware scheduler (2-D block-cyclic distribution) */
int sfx_set_home(sfx_runtime* rt, uint64_t hid, int32_t device);
int sfx_unregister(sfx_runtime* rt, uint64_t hid);

int sfx_submit(sfx_runtime* rt, uint32_t n, const sfx_task_desc* tasks, const sfx_access* accesses);
int sfx_pause(sfx_runtime* rt);
int sfx_resume(sfx_runtime* rt);
/* SFX_OK when every task of the graph completed, SFX_TIMEOUT, or an error */
int sfx_wait_all(sfx_runtime* rt, uint32_t gid, double timeout_s);
int sfx_wait_task(sfx_runtime* rt, uint64_t tid, double timeout_s);
int sfx_task_state(sfx_runtime* rt, uint64_t tid, int32_t* state);
/* insert a flush of hid to its host buffer: write_mode=1 is the reference's
 * flush_to_host (host write: device copies dropped), 0 keeps device copies */
int sfx_flush(sfx_runtime* rt, uint32_t gid, uint64_t tid, uint64_t hid, int32_t write_mode);

int sfx_stats(sfx_runtime* rt, int dev, sfx_dev_stats* out);
/* resident block handle ids of a device arena (LRU parity tests) */
int sfx_resident(sfx_runtime* rt, int dev, uint64_t* hids, uint64_t cap, uint64_t* n);
/* per-device coherency state of hid: bit0 valid, bit1 dirty; *host_valid */
int sfx_block_state(sfx_runtime* rt, uint64_t hid, int32_t dev, int32_t* state, int32_t* host_valid);
int sfx_trace(sfx_runtime* rt, uint32_t gid, sfx_event* buf, uint64_t cap, uint64_t* n);
/* successor edges of a graph: (src tid, dst tid, hid) triples, one per handle pair */
int sfx_edges(sfx_runtime* rt, uint32_t gid, uint64_t* src, uint64_t* dst, uint64_t* hid, uint64_t cap,
              uint64_t* n);
/* conflict instrumentation (handles.py:88-107): violations observed */
int sfx_violations(sfx_runtime* rt, uint64_t* n);

/* tuning knobs: "group_max" (ready same-shape tasks fused into one grouped
 * launch, default 32; 1 disables grouping), "window" (max in-flight tasks per
 * device), "groups_per_stream" (launches queued per stream, default 2),
 * "urgent_priority" (priority from which tasks use the high-priority streams,
 * default 1000000), "prefetch" (0/1: stage queued tasks' host operands while
 * all streams are busy, default 1 on CUDA), "prefetch_depth" (queued tasks
 * looked at, default 64), "kernel_timing" (0/1: launch-group timing events,
 * as SFX_FLAG_KTIME; always on while tracing), "stream_affinity" (0/1, default 1:
 * a task whose predecessor is in flight on a stream of its class is launched
 * on that stream), "deterministic" (0/1, default 0: no order-dependent FP64
 * accumulation -- the particle ops run one-sided atomic-free kernels under
 * exclusive commutative guards and no DGEMM splits K; with one stream and the
 * FIFO scheduler repeated runs are bitwise identical) */
int sfx_set_option(sfx_runtime* rt, const char* key, int64_t value);

/* external tasks (SFX_OP_EXTERN): block up to timeout_s (< 0: forever) until at
 * least one is ready, copy up to cap task ids to tids (*n = count; 0 on timeout
 * or shutdown).  The agent performs the transfer on the object's host buffer and
 * reports it with sfx_extern_done (status != 0 poisons the engine with msg). */
int sfx_extern_poll(sfx_runtime* rt, uint64_t* tids, uint64_t cap, uint64_t* n, double timeout_s);
int sfx_extern_done(sfx_runtime* rt, uint64_t tid, int status, const char* msg);
/* an external agent's failure after its task already finished (a send whose
 * payload was staged and released before the transfer): poisons the engine with
 * msg (engine.py:227-243, first failure wins) */
int sfx_fail(sfx_runtime* rt, const char* msg);

/* pinned host memory (cudaHostAlloc; aligned malloc in sim) for tiles */
int sfx_host_alloc(uint64_t bytes, int sim, void** out);
int sfx_host_free(void* p, int sim);

/* FP64 DMMA throughput microbenchmark on a device (roofline denominator) */
int sfx_fp64_peak(int ordinal, double* tflops, double* sm_mhz);
/* FP64 pipe (DFMA, 2 flop per FMA) throughput microbenchmark: the roofline
 * denominator of the particle kernel, whose work is DFMA/DMUL/DADD */
int sfx_fp64_dfma_peak(int ordinal, double* tflops);

/* DGEMM launch-path counters (process-wide, since load): which configuration of
 * the grouped DMMA kernel ran.  out[k] for k < n, n <= SFX_GEMM_PATHS.  Parity
 * tests use them to prove they exercised the benchmarked path (C-prefetch,
 * several output tiles per persistent CTA, no split-K). */
#define SFX_GEMM_LAUNCHES 0          /* grouped launches                                    */
#define SFX_GEMM_TASKS 1             /* tile tasks carried by them                          */
#define SFX_GEMM_WORK_ITEMS 2        /* (task, output tile, k-slice) work items             */
#define SFX_GEMM_CPREF 3             /* launches with the TMA C-prefetch epilogue           */
#define SFX_GEMM_MULTI_TILE 4        /* launches with >= 2 output tiles per persistent CTA  */
#define SFX_GEMM_CPREF_MULTI_TILE 5  /* both: the C2 headline configuration                 */
#define SFX_GEMM_SPLITK 6            /* split-K launches (FP64 atomic epilogue)             */
#define SFX_GEMM_TRI 7               /* TRI-masked launches (full-inverse TRSM)             */
#define SFX_GEMM_LOWER 8             /* lower-triangle launches (DSYRK)                     */
#define SFX_GEMM_NN 9                /* B stored K x N                                      */
#define SFX_GEMM_NT 10               /* B stored N x K (Cholesky update, DSYRK)             */
#define SFX_GEMM_PATHS 11
int sfx_gemm_paths(uint64_t* out, uint32_t n);

/* ---- user ops: the reference's device= callables (engine.py:144-149) ----
 * A user op is a host-side LAUNCHER the executor calls, outside the runtime
 * lock, on the thread that issues the task's stream work; it enqueues its own
 * kernels on `stream` (a cudaStream_t; NULL on the simulated backend, where
 * `data` are host pointers and the work runs synchronously).  `views` are the
 * task's accesses in declaration order, staged and pinned like the built-in
 * ops' operands -- the DeviceView of src/device.py:119-133 (device, size,
 * descriptor, data, mode).  Return 0 on success; anything else fails the task
 * and poisons the engine with SFX_ERR_USER (engine.py:154-157, 227-243).
 * The runtime waits for the stream work like any op's (end event after the
 * launcher returns), so the launcher must not synchronise. */
typedef struct sfx_view {
  void* data;           /* device pointer of the staged block                    */
  uint64_t bytes;       /* DeviceView.size                                        */
  int64_t rows, cols, ld; /* descriptor (elements; ld = row stride)                */
  int32_t dtype;        /* SFX_DTYPE_* of the registered handle                    */
  uint32_t mode;        /* SFX_READ ... of this access                             */
  int32_t device;       /* runtime device index                                    */
  int32_t reserved;
} sfx_view;
typedef int (*sfx_user_launch_fn)(const sfx_view* views, int nviews, void* stream, const double* fparam,
                                  const int64_t* iparam, void* user);
/* registers `fn` under `name` (<= 63 chars, unique) process-wide; *op gets the op
 * code to put in sfx_task_desc.op.  User ops never join launch groups. */
int sfx_register_op(const char* name, sfx_user_launch_fn fn, void* user, uint32_t* op);

#ifdef __cplusplus
}
#endif
#endif /* SFX_H */
