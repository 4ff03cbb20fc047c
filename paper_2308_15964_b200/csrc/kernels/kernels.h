// Internal launch interface of the sm_100a tile kernels (not part of the C ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "sfx.h"

namespace sfx {

// every kernel launch issued by the runtime's ops (evidence for gpu_launches)
extern std::atomic<unsigned long long> g_kernel_launches;
inline void count_launch() { g_kernel_launches.fetch_add(1, std::memory_order_relaxed); }
// DGEMM launch-path counters (SFX_GEMM_* in sfx.h)
extern std::atomic<unsigned long long> g_gemm_paths[];

// Deterministic mode (runtime option "deterministic"): set by the backend around
// a task's launches on the launching thread.  Launchers then avoid every
// order-dependent FP64 accumulation: no split-K atomics in the DGEMMs (TRSM,
// POTRF's inverse doubling included), one-sided atomic-free particle kernels.
void set_deterministic_launches(bool on);
bool deterministic_launches();

bool make_tmap_f64_2d(CUtensorMap* tm, const double* base, uint64_t inner, uint64_t outer, uint64_t ld,
                      uint32_t box_inner, uint32_t box_outer, bool swizzle128);

struct TrsmDesc {
  const double* L;
  long long ldl;
  double* B;
  long long ldb;
};

struct GemmDesc {
  const double* A;
  long long lda;
  const double* B;
  long long ldb;
  double* C;
  long long ldc;
};

// n independent same-shape GEMMs in grouped launches (up to 32 per launch)
cudaError_t launch_dgemm_group(const GemmDesc* d, int n, int M, int N, int K, double alpha, double beta,
                               bool trans_b, bool lower, cudaStream_t stream, bool tri = false);

// X L^T = B for every task, L's 64x64 diagonal blocks carrying their inverses
// (transposed, strict upper) in the upper triangle: for each 64-column panel,
// X_kb = B_kb * inv(L_kk)^T (triangular NN DMMA GEMM, in place) then
// B_j -= X_kb L_{j,kb}^T for the columns right of it (NT DMMA GEMM), all grouped
cudaError_t launch_dtrsm_inv_group(const TrsmDesc* d, int ntasks, int M, int n, cudaStream_t s);

// C = beta*C + alpha*A*op(B); op(B) = B^T ([N x K] storage) if trans_b else B ([K x N]).
// lower: only row >= col of C is computed/stored (square C).
cudaError_t launch_dgemm(const double* A, long long lda, const double* B, long long ldb, double* C, long long ldc,
                         int M, int N, int K, double alpha, double beta, bool trans_b, bool lower,
                         cudaStream_t stream);

// cooperative (single-launch) factorization kernels, n and M multiples of 64;
// workspace: per-stream scratch whose first 256 bytes are zero-initialised barrier words
size_t coop_workspace_bytes(int n);
bool coop_supported(int M, int n);
// store_inverses: also leave inv(L_jj)^T of every 64x64 diagonal block in that
// block's strict upper triangle (consumed by launch_dtrsm_inv_group)
cudaError_t launch_dpotrf_coop(double* A, long long lda, int n, int* info, void* workspace, cudaStream_t s,
                               bool store_inverses = false);
// full triangular inverse (factor_inv.cu): DPOTRF leaving inv(L)^T in the strict
// upper triangle (n = 64 * 2^k, n >= 128), and DTRSM as one TRI-masked DGEMM
bool fullinv_supported(int n);
size_t fullinv_workspace_bytes(int n);
cudaError_t launch_dpotrf_fullinv(double* A, long long lda, int n, int* info, void* workspace, size_t ws_bytes,
                                  cudaStream_t s);
// dataflow DPOTRF (potrf_flow.cu): one cooperative launch, 64x64 block tasks
// ordered by flags; store_inv 0 = LAPACK 'L', 1 = 64x64 diagonal-block inverses,
// 2 = full inv(L)^T in the strict upper triangle.  workspace: a zero-initialised
// stream scratch (the flags live at its top and are cleared by every launch)
bool flow_supported(int n);
size_t flow_workspace_bytes(int n);
cudaError_t launch_dpotrf_flow(double* A, long long lda, int n, int* info, void* workspace, size_t ws_bytes,
                               cudaStream_t s, int store_inv);
cudaError_t launch_dtrsm_fullinv(const double* L, long long ldl, double* B, long long ldb, int M, int n, void* scratch,
                                 size_t bytes, cudaStream_t s);
cudaError_t launch_dtrsm_coop_group(const TrsmDesc* d, int ntasks, int M, int n, void* workspace, size_t ws_bytes,
                                    cudaStream_t s);

cudaError_t launch_dtrsm(const double* L, long long ldl, double* B, long long ldb, int M, int n, cudaStream_t s);
// info: if non-null, receives the 1-based order of the first non-positive leading
// minor (LAPACK dpotrf info) unless it is already non-zero; `off` = column offset
cudaError_t launch_dpotrf(double* A, long long lda, int n, int* info, cudaStream_t s, int off = 0);
struct P2PDesc {
  const double* Pi;
  long long ldpi;
  int ni;
  const double* Pj;
  long long ldpj;
  int nj;
  double* Fi;
  long long ldfi;
  double* Fj;
  long long ldfj;
};
// grouped launch: tasks of one op (pair or self), one kernel per 32 tasks
cudaError_t launch_p2p_group(const P2PDesc* d, int ntasks, bool self, double eps2, cudaStream_t s);
cudaError_t launch_p2p(const double* Pi, long long ldpi, int ni, const double* Pj, long long ldpj, int nj, double* Fi,
                       long long ldfi, double* Fj, long long ldfj, bool self, double eps2, cudaStream_t s);

cudaError_t launch_fill_uniform(double* a, long long rows, long long cols, long long ld, long long seed,
                                long long row0, long long col0, long long ncols_total, cudaStream_t s);
cudaError_t launch_fill_spd(double* a, long long rows, long long cols, long long ld, long long seed, long long row0,
                            long long col0, long long n, cudaStream_t s);
cudaError_t launch_fill_particles(double* p, long long n, long long ld, long long seed, long long first,
                                  cudaStream_t s);
cudaError_t launch_spin(long long ns, cudaStream_t s);
cudaError_t launch_spin_group(int n, long long ns, cudaStream_t s);
// failure injection (SFX_OP_FAULT): 0 = invalid launch configuration, 1 = device trap
cudaError_t launch_fault(int kind, cudaStream_t s);
// A += sum of n addends (FP64 rows x cols, each with its own ld), n <= 7
cudaError_t launch_dacc(double* a, long long lda, long long rows, long long cols, const double* const* add,
                        const long long* ld, int n, cudaStream_t s);
cudaError_t launch_add_i64(long long* const* cells, int n, long long delta, cudaStream_t s);
cudaError_t launch_cell(long long* target, const long long* const* reads, int nreads, long long kind, long long a,
                        long long b, cudaStream_t s);
cudaError_t launch_bytes_add(unsigned char* p, long long off, long long len, long long delta, cudaStream_t s);
cudaError_t fp64_dmma_peak(int iters, double* tflops);
cudaError_t fp64_dfma_peak(int iters, double* tflops);

}  // namespace sfx
