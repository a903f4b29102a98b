/* cclp_cu — B200-native PDHG engine behind the reference's run_pdhg interface.
 *
 * C ABI (plain pointers and sizes, no C++/torch types) exported by
 * paper_2510_24429_b200/libcclp_cuda.so. It replaces the reference's hot path
 *
 *   cclp::run_pdhg(const LinearProgram&, const PdhgConfig&, const Tolerances&,
 *                  const std::vector<Scalar>& thresholds, const SnapshotSink&,
 *                  const std::atomic<bool>* cancel) -> PdhgResult
 *   (reference: proj/include/cclp/pdhg.hpp:138-142, proj/src/pdhg.cpp:230-378)
 *
 * and the kernels it is built from (matvec / matvec_transpose,
 * kernels.hpp:27-40; ruiz_scale, scaling.hpp:47-48; estimate_matrix_norm,
 * pdhg.hpp:85-86). A C++ drop-in that re-implements cclp::run_pdhg on top of
 * this ABI is shown in INTEGRATION.md.
 *
 * Conventions (mirroring the reference):
 *  - The LP is equality form, CSC exactly as Eigen stores a compressed
 *    SparseMatrix<double, ColMajor, int> (types.hpp:31): colptr = outerIndexPtr,
 *    rowind = innerIndexPtr (ascending per column), val = valuePtr; bounds use
 *    IEEE +-inf (types.hpp:35).
 *  - Return codes: 0 ok; CCLP_CU_EINVAL where the reference throws
 *    std::invalid_argument (pdhg.cpp:235-244); CCLP_CU_ECUDA / CCLP_CU_ENOMEM on
 *    device failure. A non-finite iterate is NOT an error: it is stop reason
 *    CCLP_CU_STOP_NUMERICAL_ERROR with error_iteration set (pdhg.cpp:369-376).
 *  - The snapshot sink runs on the calling thread with pointers valid only
 *    for the duration of the call (pdhg.cpp:346-358). The snapshot is the
 *    reference's (same iterate, threshold, maxresid, iteration); it is taken
 *    by the iteration kernels into a device slot and copied out on a side
 *    stream, so the device keeps iterating while the sink runs.
 *  - cancel is polled every iteration (pdhg.cpp:301): the host loop mirrors
 *    the caller's byte into device-mapped memory that the kernels read, so the
 *    loop stops within one iteration of the host seeing the flag.
 *  - One context per host thread; a context is not thread-safe (except
 *    cclp_cu_request_cancel).
 */
#ifndef CCLP_CU_H_
#define CCLP_CU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CCLP_CU_OK 0
#define CCLP_CU_EINVAL 1
#define CCLP_CU_ECUDA 2
#define CCLP_CU_ENOMEM 3
#define CCLP_CU_ENCCL 4

/* PdhgStopReason (pdhg.hpp:44-51), same order. */
#define CCLP_CU_STOP_CONVERGED 0
#define CCLP_CU_STOP_ITERATION_LIMIT 1
#define CCLP_CU_STOP_TIME_LIMIT 2
#define CCLP_CU_STOP_CANCELLED 3
#define CCLP_CU_STOP_WON_BY_CROSSOVER 4
#define CCLP_CU_STOP_NUMERICAL_ERROR 5

/* LinearProgram (lp.hpp:37-64), the fields run_pdhg reads. */
typedef struct {
  int32_t m, n;
  const int32_t* colptr; /* n+1 */
  const int32_t* rowind; /* colptr[n] */
  const double* val;     /* colptr[n] */
  const double* c;         /* n */
  const double* row_lower; /* m */
  const double* row_upper; /* m */
  const double* col_lower; /* n */
  const double* col_upper; /* n */
} cclp_cu_lp;

/* PdhgConfig (pdhg.hpp:29-42) plus the engine's own knobs (last two). */
typedef struct {
  double step_scale;      /* eta, 0.9 */
  double primal_weight;   /* omega; <= 0 picks ||c'||/||b'|| */
  double restart_factor;  /* 0.5 */
  double time_limit;      /* seconds, +inf */
  int32_t norm_iterations;    /* 100 */
  int32_t scaling_iterations; /* 10 */
  int64_t max_iterations;     /* 2e6 */
  int32_t check_interval;     /* 1 */
  uint64_t seed;              /* 0 */
  int64_t log_interval;       /* 0 disables the iteration log */
  int32_t deterministic;      /* always honoured: fixed reduction order */
  int32_t poll_interval;      /* iterations per device batch (0 -> 64) */
  int32_t exact_spmv;         /* 1: every SpMV row sum in the reference's own
                                 sequential order (bit-identical products;
                                 slower on long rows). 0: G lanes per row with
                                 a fixed butterfly (deterministic). */
} cclp_cu_config;

/* Tolerances (kkt.hpp:32-41). */
typedef struct {
  double eps_rel, eps_abs, eps_cross, decrement;
} cclp_cu_tolerances;

/* ResidualReport (kkt.hpp:43-58), same field order. */
typedef struct {
  double rp_norm2, rd_norm2, rp_inf, rd_inf;
  double primal_objective, dual_objective, gap_abs;
  double rel_primal, rel_dual, rel_gap, maxresid_rel, complementarity;
} cclp_cu_report;

/* PdhgSnapshot (pdhg.hpp:111-117). Arrays valid only during the sink call. */
typedef struct {
  const double* x; /* n, unscaled standard-form */
  const double* y; /* m */
  const double* z; /* n */
  int32_t m, n;
  double threshold;
  double maxresid;
  int32_t from_average;
  int64_t iteration;
} cclp_cu_snapshot;

typedef void (*cclp_cu_sink_fn)(const cclp_cu_snapshot* snap, void* user);
/* One iteration-log line in the reference's format (pdhg.cpp:332-340). */
typedef void (*cclp_cu_log_fn)(const char* line, void* user);

/* PdhgResult (pdhg.hpp:121-129) plus engine timings. */
typedef struct {
  int32_t stop;
  int64_t iterations;
  int64_t restarts;
  int64_t error_iteration;
  double seconds;
  cclp_cu_report report;
  double norm_estimate, omega, tau, sigma;
  double setup_seconds; /* upload excluded: scaling + norm + init */
  double loop_seconds;  /* device time of the iteration loop */
  int64_t kernel_launches;
} cclp_cu_result;

typedef struct cclp_cu_ctx cclp_cu_ctx;

const char* cclp_cu_last_error(void);
const char* cclp_cu_stop_string(int32_t stop); /* to_string, pdhg.cpp:28-44 */
void cclp_cu_default_config(cclp_cu_config* cfg);      /* pdhg.hpp:29-42 */
void cclp_cu_default_tolerances(cclp_cu_tolerances* t); /* kkt.hpp:33-36 */

/* Uploads the CSC and bounds to `device` and builds CSR(A) on the device. */
int cclp_cu_create(const cclp_cu_lp* lp, int device, cclp_cu_ctx** out);
/* LP ingest from a binary CSC file (layout in paper_2510_24429_b200/lp.py,
 * magic "CCLPCSC1"): the file is memory-mapped and streamed to the device
 * through the multi-threaded pinned staging, then as cclp_cu_create.
 * m_out / n_out (optional) receive the dimensions. */
int cclp_cu_create_from_file(const char* path, int device, cclp_cu_ctx** out, int32_t* m_out,
                             int32_t* n_out);
int cclp_cu_destroy(cclp_cu_ctx* ctx);

/* run_pdhg on a context (pdhg.cpp:230-378): Ruiz scaling, ||A|| estimate,
 * the fused iteration loop, ladder snapshots, result download.
 * x_out/z_out: n doubles, y_out: m doubles (host). log may be NULL. */
int cclp_cu_solve(cclp_cu_ctx* ctx, const cclp_cu_config* cfg, const cclp_cu_tolerances* tol,
                  const double* thresholds, int32_t nthr, cclp_cu_sink_fn sink, void* sink_user,
                  const volatile uint8_t* cancel, cclp_cu_log_fn log, void* log_user,
                  double* x_out, double* y_out, double* z_out, cclp_cu_result* res);

/* Asks a running cclp_cu_solve on `ctx` to stop (stop reason CANCELLED) at
 * the next iteration, exactly as setting its cancel byte would. Safe to call
 * from any thread, including from inside the snapshot sink (the C++ drop-in
 * uses it to stop the loop when the sink throws, then rethrows). */
int cclp_cu_request_cancel(cclp_cu_ctx* ctx);

/* One-shot drop-in: create + solve + destroy. */
int cclp_cu_run_pdhg(const cclp_cu_lp* lp, const cclp_cu_config* cfg, const cclp_cu_tolerances* tol,
                     const double* thresholds, int32_t nthr, cclp_cu_sink_fn sink, void* sink_user,
                     const volatile uint8_t* cancel, double* x_out, double* y_out, double* z_out,
                     cclp_cu_result* res, int device);

/* ---- kernel-level entry points (unscaled A held by the context) ---------- */

/* matvec / matvec_transpose (kernels.hpp:27-40). Host in, host out. */
int cclp_cu_matvec(cclp_cu_ctx* ctx, const double* x, double* out);
int cclp_cu_matvec_transpose(cclp_cu_ctx* ctx, const double* y, double* out);
/* relative_report and absolute_violation (kkt.hpp:76,84; kkt.cpp:106-149) of
 * the iterate (x[n], y[m], z[n]) on the context's unscaled LP, which must be
 * in equality form (as run_pdhg requires). abs_violation may be NULL. Sums are
 * reduced in a fixed order (within rounding of the reference's); maxima exact. */
int cclp_cu_relative_report(cclp_cu_ctx* ctx, const double* x, const double* y, const double* z,
                            cclp_cu_report* out, double* abs_violation);
/* Crossover pricing (simplex.cpp:266-296, price()) on the device for the
 * EngineModel of the context's equality-form LP: n structural columns then
 * m logical ones (basis.hpp:30-58). status[n+m] holds ColStatus chars
 * ('B','L','U','X','Z'), skip[n+m] (optional) nonzero for the skip set,
 * y[m] the duals. d_j = cost_j - column_dot(j, y) in column_dot's own order;
 * returns the reference's pick: entering column (-1: none), direction (+1 /
 * -1) and violation (Dantzig: largest, first index on ties; bland != 0:
 * first violating index). */
int cclp_cu_price(cclp_cu_ctx* ctx, const double* y, const char* status, const uint8_t* skip, int32_t phase1,
                  double dtol, int32_t bland, int64_t* entering, int32_t* direction, double* violation);
/* ruiz_scale factors (scaling.cpp:46-90): row_scale[m], col_scale[n]. */
int cclp_cu_ruiz(cclp_cu_ctx* ctx, int32_t iterations, double* row_scale, double* col_scale);
/* estimate_matrix_norm (pdhg.cpp:46-65) on the unscaled A. */
int cclp_cu_estimate_norm(cclp_cu_ctx* ctx, int32_t iterations, uint64_t seed, double* out);

/* The power iteration's start vector (host only, no device needed):
 * out[j] = std::normal_distribution<double>(0,1) draws from
 * std::mt19937_64(seed + 0x9e3779b97f4a7c15), pdhg.cpp:49-52, bit for bit. */
void cclp_cu_gaussian_start(uint64_t seed, int64_t n, double* out);

/* ---- measurement hooks (bench.py) ---------------------------------------- */

/* Begin a solve without running the loop: scaling, norm, initial check. */
int cclp_cu_begin(cclp_cu_ctx* ctx, const cclp_cu_config* cfg, const cclp_cu_tolerances* tol);
/* Advance exactly `iters` PDHG iterations (ignoring convergence and the
 * iteration limit) with the full per-iteration checks, timed with CUDA
 * events on the engine stream; returns device milliseconds. */
int cclp_cu_advance(cclp_cu_ctx* ctx, int64_t iters, double* device_ms);
/* Per-kernel device time: runs `iters` iterations launching kernels eagerly
 * with events between them; out[0..3] = average ms of k_spmv_rows (A x),
 * k_dual (dual update + row reports), k_spmv_cols (A'y) and k_primal (primal
 * update + column reports + candidates + on-device decisions). */
int cclp_cu_profile_kernels(cclp_cu_ctx* ctx, int64_t iters, double* out);
/* The same split as it runs inside the CUDA graphs of the loop: block 0 of
 * each kernel stamps %globaltimer after its PDL wait (= the previous kernel's
 * completion), over the last 128 steps; out[0..3] = median microseconds of
 * rows / dual / cols / primal+decisions per step, *steps = steps used.
 * Single-device contexts after cclp_cu_begin/cclp_cu_advance. */
int cclp_cu_phase_profile(cclp_cu_ctx* ctx, double* out, int64_t* steps);
/* The engine's CUDA stream (cudaStream_t) for external event timing. */
void* cclp_cu_stream(cclp_cu_ctx* ctx);
/* Static description: nnz, CSR/CSC group sizes, grid sizes, bytes/iteration. */
int cclp_cu_describe(cclp_cu_ctx* ctx, int64_t* out, int32_t nout);

/* ---- sharded solve: row-block partition over several GPUs --
 * A is split by rows and A' (the CSC) by columns into P nnz-balanced blocks;
 * each shard computes its rows of A x and A' y completely (no cross-shard
 * sums: iterates bit-identical to one GPU) and all-gathers y, the 22 report
 * sums and x once per iteration. Two transports behind one API:
 *   nccl_id NULL: `nshards` shards in this process on `device`, exchanging
 *                by device copies (development and tests on one GPU);
 *   nccl_id set: NCCL, this process is `rank` of `nranks` (one GPU each,
 *                nshards = 1); `nccl_id` = the 128-byte id from
 *                cclp_cu_nccl_unique_id on rank 0, broadcast by the caller
 *                (nranks may be 1: the collective path on one GPU).
 * Every rank passes the full LP and receives the full result. The run_pdhg
 * setup (Ruiz, ||A||) is replicated per rank; the iteration is sharded.
 * Exchanges: by default (P <= 8) stores fused into the producing kernels
 * plus epoch flags (CUDA IPC peers across processes, opened at setup); with
 * CCLP_CU_TRANSPORT=gather, device copies in-process or NCCL all-gathers /
 * halo send/recv across processes. */
typedef struct cclp_cu_sharded cclp_cu_sharded;
int cclp_cu_nccl_unique_id(uint8_t* out128);
int cclp_cu_sharded_create(const cclp_cu_lp* lp, int device, int32_t nshards, int32_t rank,
                           int32_t nranks, const uint8_t* nccl_id, cclp_cu_sharded** out);
int cclp_cu_sharded_solve(cclp_cu_sharded* ctx, const cclp_cu_config* cfg,
                          const cclp_cu_tolerances* tol, const double* thresholds, int32_t nthr,
                          cclp_cu_sink_fn sink, void* sink_user, const volatile uint8_t* cancel,
                          double* x_out, double* y_out, double* z_out, cclp_cu_result* res);
/* Multi-process without NCCL: the caller provides an all-gather of host
 * bytes (e.g. over its own MPI / gloo); the iteration then runs the push
 * transport over CUDA IPC (P <= 8 ranks, one shard each). */
typedef struct {
  /* in: `bytes` from this rank; out: nranks * bytes, rank order; 0 = ok */
  int (*allgather)(const void* in, size_t bytes, void* out, void* user);
  void* user;
} cclp_cu_host_comm;
int cclp_cu_sharded_create_hostcomm(const cclp_cu_lp* lp, int device, int32_t rank, int32_t nranks,
                                    const cclp_cu_host_comm* comm, cclp_cu_sharded** out);
/* measurement hooks, as cclp_cu_begin / cclp_cu_advance */
int cclp_cu_sharded_begin(cclp_cu_sharded* ctx, const cclp_cu_config* cfg,
                          const cclp_cu_tolerances* tol);
int cclp_cu_sharded_advance(cclp_cu_sharded* ctx, int64_t iters, double* device_ms);
/* out: P, row bounds [P+1], column bounds [P+1], launches, then for the x
 * and y exchanges: halo on (1) or all-gather (0), and the halo volume in
 * doubles per iteration summed over shards */
int cclp_cu_sharded_describe(cclp_cu_sharded* ctx, int64_t* out, int32_t nout);
int cclp_cu_sharded_destroy(cclp_cu_sharded* ctx);
/* As cclp_cu_request_cancel for a running cclp_cu_sharded_solve (seen at the
 * next batch boundary, agreed by every rank). */
int cclp_cu_sharded_request_cancel(cclp_cu_sharded* ctx);
/* The nnz-balanced split used for the shards (host only): part b starts at
 * the first i with ptr[i] + 4 i >= (ptr[rows] + 4 rows) b / parts. */
int cclp_cu_partition(const int32_t* ptr, int32_t rows, int32_t parts, int32_t* bounds);

#ifdef __cplusplus
}
#endif

#endif /* CCLP_CU_H_ */
