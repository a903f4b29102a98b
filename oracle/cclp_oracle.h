/* CPU restatement of the reference PDHG path — TEST INFRASTRUCTURE ONLY.
 *
 * Plain C11 restatement of cclp::run_pdhg and the helpers it calls
 * (reference: /root/reference/proj/src/pdhg.cpp, scaling.cpp, kkt.cpp,
 * lp.cpp). It is the checker for the CUDA engine: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it. It is
 * pinned against the reference itself (oracle/_ref, built from the reference's
 * own sources) and the golden fixtures in tests/golden/.
 *
 * Arithmetic follows the reference build (x86-64, SSE2, no FMA contraction;
 * compiled here with -ffp-contract=off): Eigen's column-scatter A*x and
 * per-column gather A'y, Eigen's 2x2-packet redux order for dot()/norm(),
 * plain sequential loops where the reference loops.
 */
#ifndef CCLP_ORACLE_H_
#define CCLP_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Equality-form LP in the reference's layout: CSC A (types.hpp:31), int32
 * indices, fp64 values; row_lower/row_upper (equal in equality form),
 * col_lower/col_upper with +-inf for absent bounds (types.hpp:35). */
typedef struct {
  int m, n;
  const int* colptr; /* n+1 */
  const int* rowind; /* nnz, ascending within a column */
  const double* val; /* nnz */
  const double* c;
  const double* row_lower;
  const double* row_upper;
  const double* col_lower;
  const double* col_upper;
} oracle_lp;

/* PdhgConfig (pdhg.hpp:29-42). */
typedef struct {
  double step_scale;     /* 0.9 */
  double primal_weight;  /* 0 -> ||c'||/||b'|| */
  double restart_factor; /* 0.5 */
  double time_limit;     /* seconds, +inf */
  int norm_iterations;   /* 100 */
  int scaling_iterations;/* 10 */
  int64_t max_iterations;/* 2e6 */
  int check_interval;    /* 1 */
  uint64_t seed;         /* 0 */
} oracle_config;

/* Tolerances (kkt.hpp:32-41). */
typedef struct {
  double eps_rel, eps_abs, eps_cross, decrement;
} oracle_tol;

/* ResidualReport (kkt.hpp:43-58), same field order. */
typedef struct {
  double rp_norm2, rd_norm2, rp_inf, rd_inf;
  double primal_objective, dual_objective, gap_abs;
  double rel_primal, rel_dual, rel_gap, maxresid_rel, complementarity;
} oracle_report;

/* PdhgStopReason (pdhg.hpp:44-51). */
enum {
  ORACLE_CONVERGED = 0,
  ORACLE_ITERATION_LIMIT = 1,
  ORACLE_TIME_LIMIT = 2,
  ORACLE_CANCELLED = 3,
  ORACLE_WON_BY_CROSSOVER = 4,
  ORACLE_NUMERICAL_ERROR = 5
};

typedef struct {
  double threshold, maxresid;
  int from_average;
  int64_t iteration;
  const double *x, *y, *z; /* valid only during the callback */
} oracle_snapshot;

typedef void (*oracle_sink)(const oracle_snapshot* snap, void* user);

typedef struct {
  int stop;
  int64_t iterations, restarts, error_iteration;
  double seconds;
  oracle_report report;
  double tau, sigma, norm_estimate, omega;
} oracle_result;

/* Optional instrumentation (not in the reference API): restart iterations and
 * a per-check trace of (iteration, cur maxresid, avg maxresid or -1). */
typedef struct {
  int64_t* restart_iters;
  int64_t restart_cap;
  int64_t n_restarts_logged;
  double* trace; /* 3 doubles per check */
  int64_t trace_cap;
  int64_t n_trace;
} oracle_trace;

void oracle_defaults(oracle_config* cfg, oracle_tol* tol);

/* A*x (Eigen ColMajor scatter) and A'*y (per-column gather). */
void oracle_matvec(const oracle_lp* lp, const double* x, double* out);
void oracle_matvec_transpose(const oracle_lp* lp, const double* y, double* out);

/* Eigen 3.4 redux order for dot() and norm(). */
double oracle_dot(const double* a, const double* b, int64_t n);
double oracle_norm(const double* a, int64_t n);

/* pow2_sqrt (scaling.cpp:23-25). */
double oracle_pow2_sqrt(double v);

/* Ruiz factors (scaling.cpp:46-90) and the scaled values (apply_scaling
 * scaling.cpp:29-44): row_scale[m], col_scale[n], scaled_val[nnz] (nullable). */
void oracle_ruiz(const oracle_lp* lp, int iterations, double* row_scale, double* col_scale,
                 double* scaled_val);

/* Standard-normal start vector of estimate_matrix_norm (pdhg.cpp:49-54):
 * mt19937_64(seed + 0x9e3779b97f4a7c15) fed through libstdc++'s
 * normal_distribution (Marsaglia polar, second value cached). */
void oracle_gaussian_start(uint64_t seed, int64_t n, double* v);

/* estimate_matrix_norm (pdhg.cpp:46-65). */
double oracle_estimate_norm(const oracle_lp* lp, int iterations, uint64_t seed);

/* relative_report (kkt.cpp:119-139): independent re-verification with fresh
 * matvecs. */
void oracle_relative_report(const oracle_lp* lp, const double* x, const double* y, const double* z,
                            oracle_report* rep);

/* run_pdhg (pdhg.cpp:230-378). Returns 0, or 1 on invalid arguments (the
 * reference's std::invalid_argument), with a message in oracle_last_error().
 * x_out/z_out: n, y_out: m (unscaled standard-form iterate). cancel: nullable
 * flag polled every pass. trace: nullable. */
int oracle_run_pdhg(const oracle_lp* lp, const oracle_config* cfg, const oracle_tol* tol,
                    const double* thresholds, int nthr, oracle_sink sink, void* sink_user,
                    const volatile uint8_t* cancel, double* x_out, double* y_out, double* z_out,
                    oracle_result* res, oracle_trace* trace);

const char* oracle_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* CCLP_ORACLE_H_ */
