/* CPU restatement of the reference PDHG path — TEST INFRASTRUCTURE ONLY.
 * See cclp_oracle.h. Every function cites the reference file:line it
 * restates (paths relative to /root/reference/proj/). */
#define _POSIX_C_SOURCE 200809L
#include "cclp_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static char g_err[256];
const char* oracle_last_error(void) { return g_err; }

/* std::max / std::min semantics (first argument wins ties / NaN). */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }
/* cclp::is_finite (types.hpp:37). */
static inline int is_fin(double v) { return v > -INFINITY && v < INFINITY; }

void oracle_defaults(oracle_config* cfg, oracle_tol* tol) {
  /* pdhg.hpp:29-42, kkt.hpp:32-36 */
  if (cfg) {
    cfg->step_scale = 0.9;
    cfg->primal_weight = 0.0;
    cfg->restart_factor = 0.5;
    cfg->time_limit = INFINITY;
    cfg->norm_iterations = 100;
    cfg->scaling_iterations = 10;
    cfg->max_iterations = 2000000;
    cfg->check_interval = 1;
    cfg->seed = 0;
  }
  if (tol) {
    tol->eps_rel = 1e-6;
    tol->eps_abs = 1e-6;
    tol->eps_cross = 1e-2;
    tol->decrement = 0.1;
  }
}

/* ---- Eigen semantics --------------------------------------------------- */

/* Eigen 3.4 Redux.h LinearVectorizedTraversal with 2-wide SSE2 packets:
 * accumulators p0=(e0,e1), p1=(e2,e3), strided by 4; p0+=p1; one extra
 * aligned pair; horizontal add; odd tail. */
#define REDUX_BODY(COEFF)                                                  \
  if (n == 0) return 0.0;                                                  \
  const int64_t aligned2 = (n / 4) * 4, aligned = (n / 2) * 2;             \
  double res;                                                              \
  if (aligned) {                                                           \
    int64_t i = 0;                                                         \
    double p0a, p0b;                                                       \
    i = 0; p0a = COEFF; i = 1; p0b = COEFF;                                \
    if (aligned > 2) {                                                     \
      double p1a, p1b;                                                     \
      i = 2; p1a = COEFF; i = 3; p1b = COEFF;                              \
      for (int64_t k = 4; k < aligned2; k += 4) {                          \
        i = k; p0a = p0a + (COEFF);                                        \
        i = k + 1; p0b = p0b + (COEFF);                                    \
        i = k + 2; p1a = p1a + (COEFF);                                    \
        i = k + 3; p1b = p1b + (COEFF);                                    \
      }                                                                    \
      p0a = p0a + p1a;                                                     \
      p0b = p0b + p1b;                                                     \
      if (aligned > aligned2) {                                            \
        i = aligned2; p0a = p0a + (COEFF);                                 \
        i = aligned2 + 1; p0b = p0b + (COEFF);                             \
      }                                                                    \
    }                                                                      \
    res = p0a + p0b;                                                       \
    for (i = aligned; i < n; ++i) res = res + (COEFF);                     \
  } else {                                                                 \
    int64_t i = 0;                                                         \
    res = COEFF;                                                           \
    for (i = 1; i < n; ++i) res = res + (COEFF);                           \
  }                                                                        \
  return res;

double oracle_dot(const double* a, const double* b, int64_t n) { REDUX_BODY(a[i] * b[i]) }
static double sq_sum(const double* a, int64_t n) { REDUX_BODY(a[i] * a[i]) }
double oracle_norm(const double* a, int64_t n) { return sqrt(sq_sum(a, n)); }

/* A*x: Eigen ColMajor sparse*dense (dst.setZero(); res[i] += a_ij * (1*x_j)
 * in ascending j) — the call sites are pdhg.cpp:57,113,124. */
void oracle_matvec(const oracle_lp* lp, const double* x, double* out) {
  for (int i = 0; i < lp->m; ++i) out[i] = 0.0;
  for (int j = 0; j < lp->n; ++j) {
    const double xj = 1.0 * x[j];
    for (int p = lp->colptr[j]; p < lp->colptr[j + 1]; ++p) out[lp->rowind[p]] += lp->val[p] * xj;
  }
}

/* A'*y: Eigen RowMajor (transposed view) processRow: tmp = sum a_ij*y_i in
 * ascending i, res_j = 0 + 1*tmp — pdhg.cpp:58,114,127. */
void oracle_matvec_transpose(const oracle_lp* lp, const double* y, double* out) {
  for (int j = 0; j < lp->n; ++j) {
    double tmp = 0.0;
    for (int p = lp->colptr[j]; p < lp->colptr[j + 1]; ++p) tmp += lp->val[p] * y[lp->rowind[p]];
    out[j] = 0.0 + 1.0 * tmp;
  }
}

/* ---- scaling.cpp ------------------------------------------------------- */

double oracle_pow2_sqrt(double v) { return exp2(round(0.5 * log2(v))); } /* scaling.cpp:23-25 */

void oracle_ruiz(const oracle_lp* lp, int iterations, double* r, double* s, double* scaled_val) {
  const int m = lp->m, n = lp->n;
  double* row_max = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  double* col_max = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (int i = 0; i < m; ++i) r[i] = 1.0; /* scaling.cpp:51-52 */
  for (int j = 0; j < n; ++j) s[j] = 1.0;
  for (int t = 0; t < iterations; ++t) { /* scaling.cpp:55-88 */
    for (int i = 0; i < m; ++i) row_max[i] = 0.0;
    for (int j = 0; j < n; ++j) col_max[j] = 0.0;
    for (int j = 0; j < n; ++j) {
      for (int p = lp->colptr[j]; p < lp->colptr[j + 1]; ++p) {
        const int i = lp->rowind[p];
        const double v = fabs(lp->val[p]) * r[i] * s[j];
        if (v > row_max[i]) row_max[i] = v;
        if (v > col_max[j]) col_max[j] = v;
      }
    }
    int done = 1;
    for (int i = 0; i < m && done; ++i)
      if (row_max[i] > 0.0 && (row_max[i] < 0.5 || row_max[i] >= 2.0)) done = 0;
    for (int j = 0; j < n && done; ++j)
      if (col_max[j] > 0.0 && (col_max[j] < 0.5 || col_max[j] >= 2.0)) done = 0;
    if (done) break;
    for (int i = 0; i < m; ++i)
      if (row_max[i] > 0.0) r[i] /= oracle_pow2_sqrt(row_max[i]);
    for (int j = 0; j < n; ++j)
      if (col_max[j] > 0.0) s[j] /= oracle_pow2_sqrt(col_max[j]);
  }
  if (scaled_val) { /* apply_scaling, scaling.cpp:33-37 */
    for (int j = 0; j < n; ++j)
      for (int p = lp->colptr[j]; p < lp->colptr[j + 1]; ++p)
        scaled_val[p] = lp->val[p] * (r[lp->rowind[p]] * s[j]);
  }
  free(row_max);
  free(col_max);
}

/* ---- estimate_matrix_norm (pdhg.cpp:46-65) ----------------------------- */

typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int k = 0; k < 312; ++k) {
      const uint64_t y = (g->mt[k] & upper) | (g->mt[(k + 1) % 312] & lower);
      g->mt[k] = g->mt[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    }
    g->idx = 0;
  }
  uint64_t z = g->mt[g->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

/* libstdc++ generate_canonical<double, 53>(mt19937_64): one draw, u / 2^64. */
static double canonical(mt64* g) {
  double ret = (double)mt64_next(g) / 18446744073709551616.0;
  if (ret >= 1.0) ret = nextafter(1.0, 0.0);
  return ret;
}

void oracle_gaussian_start(uint64_t seed, int64_t n, double* v) {
  mt64 g;
  mt64_seed(&g, seed + 0x9e3779b97f4a7c15ULL);
  int have_saved = 0;
  double saved = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    double ret;
    if (have_saved) {
      have_saved = 0;
      ret = saved;
    } else {
      double x, y, r2;
      do {
        x = 2.0 * canonical(&g) - 1.0;
        y = 2.0 * canonical(&g) - 1.0;
        r2 = x * x + y * y;
      } while (r2 > 1.0 || r2 == 0.0);
      const double mult = sqrt(-2 * log(r2) / r2);
      saved = x * mult;
      have_saved = 1;
      ret = y * mult;
    }
    v[j] = ret * 1.0 + 0.0;
  }
}

double oracle_estimate_norm(const oracle_lp* lp, int iterations, uint64_t seed) {
  const int m = lp->m, n = lp->n;
  if (m == 0 || n == 0 || lp->colptr[n] == 0) return 0.0;
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  double* u = (double*)malloc(sizeof(double) * (size_t)n);
  double* w = (double*)malloc(sizeof(double) * (size_t)m);
  oracle_gaussian_start(seed, n, v);
  if (oracle_norm(v, n) == 0.0)
    for (int j = 0; j < n; ++j) v[j] = 1.0;
  {
    const double nv = oracle_norm(v, n);
    for (int j = 0; j < n; ++j) v[j] = v[j] / nv;
  }
  double lambda = 0.0, out = -1.0;
  for (int t = 0; t < iterations; ++t) {
    oracle_matvec(lp, v, w);
    oracle_matvec_transpose(lp, w, u);
    const double nu = oracle_norm(u, n);
    if (nu == 0.0) {
      out = 0.0;
      break;
    }
    lambda = oracle_dot(v, u, n);
    for (int j = 0; j < n; ++j) v[j] = u[j] / nu;
  }
  if (out < 0.0) out = sqrt(smax(lambda, 0.0));
  free(v);
  free(u);
  free(w);
  return out;
}

/* ---- kkt.cpp / pdhg.cpp reports --------------------------------------- */

/* clipped_reduced_costs (pdhg.cpp:89-108). */
static void clipped_z(const oracle_lp* lp, const double* x, const double* aty, double* z) {
  for (int j = 0; j < lp->n; ++j) {
    double zj = lp->c[j] - aty[j];
    const double l = lp->col_lower[j], u = lp->col_upper[j];
    const int lo = is_fin(l), up = is_fin(u);
    if (!lo && !up) {
      zj = 0.0;
    } else if (lo && up) {
      const double dl = x[j] - l, du = u - x[j];
      zj = dl <= du ? smax(zj, 0.0) : smin(zj, 0.0);
    } else if (lo) {
      zj = smax(zj, 0.0);
    } else {
      zj = smin(zj, 0.0);
    }
    z[j] = zj;
  }
}

static double max3(double a, double b, double c) { /* std::max({a,b,c}) */
  double r = a;
  if (r < b) r = b;
  if (r < c) r = c;
  return r;
}

/* report_from_products (pdhg.cpp:170-220). */
static void report_from_products(const oracle_lp* lp, const double* x, const double* y,
                                 const double* z, const double* ax, const double* aty,
                                 double b_norm, double c_norm, oracle_report* rep) {
  double rp2 = 0.0, rp_inf = 0.0;
  for (int i = 0; i < lp->m; ++i) {
    double v = 0.0;
    if (ax[i] < lp->row_lower[i]) {
      v = lp->row_lower[i] - ax[i];
    } else if (ax[i] > lp->row_upper[i]) {
      v = ax[i] - lp->row_upper[i];
    }
    rp2 += v * v;
    rp_inf = smax(rp_inf, v);
  }
  double rd2 = 0.0, rd_inf = 0.0, compl_inf = 0.0, dbt = 0.0;
  for (int j = 0; j < lp->n; ++j) {
    const double l = lp->col_lower[j], u = lp->col_upper[j];
    const double rd = aty[j] + z[j] - lp->c[j];
    rd2 += rd * rd;
    rd_inf = smax(rd_inf, fabs(rd));
    const double bv = max3(l - x[j], x[j] - u, 0.0);
    rp_inf = smax(rp_inf, bv);
    double dist = INFINITY;
    if (is_fin(l)) dist = smin(dist, fabs(x[j] - l));
    if (is_fin(u)) dist = smin(dist, fabs(x[j] - u));
    if (is_fin(dist)) compl_inf = smax(compl_inf, dist * fabs(z[j]));
    if (z[j] > 0.0 && is_fin(l)) {
      dbt += l * z[j];
    } else if (z[j] < 0.0 && is_fin(u)) {
      dbt += u * z[j];
    }
  }
  rep->rp_norm2 = sqrt(rp2);
  rep->rd_norm2 = sqrt(rd2);
  rep->rp_inf = rp_inf;
  rep->rd_inf = rd_inf;
  rep->complementarity = compl_inf;
  rep->primal_objective = oracle_dot(lp->c, x, lp->n);
  rep->dual_objective = oracle_dot(lp->row_lower, y, lp->m) + dbt;
  rep->gap_abs = fabs(rep->primal_objective - rep->dual_objective);
  rep->rel_primal = rep->rp_norm2 / (1.0 + b_norm);
  rep->rel_dual = rep->rd_norm2 / (1.0 + c_norm);
  rep->rel_gap = rep->gap_abs / (1.0 + fabs(rep->primal_objective) + fabs(rep->dual_objective));
  rep->maxresid_rel = max3(rep->rel_primal, rep->rel_dual, rep->rel_gap);
}

/* representative_rhs (lp.cpp:29-39). */
static void representative_rhs(const oracle_lp* lp, double* b) {
  for (int i = 0; i < lp->m; ++i) {
    b[i] = 0.0;
    if (is_fin(lp->row_upper[i]))
      b[i] = lp->row_upper[i];
    else if (is_fin(lp->row_lower[i]))
      b[i] = lp->row_lower[i];
  }
}

/* relative_report (kkt.cpp:119-139), with primal_residual (:50-68),
 * bound_violations (:70-78), dual_residual (:80-83), objective_gap (:85-99),
 * complementarity_inf (:103-117). */
void oracle_relative_report(const oracle_lp* lp, const double* x, const double* y, const double* z,
                            oracle_report* rep) {
  const int m = lp->m, n = lp->n;
  double* ax = (double*)malloc(sizeof(double) * (size_t)(m + 1));
  double* rp = (double*)malloc(sizeof(double) * (size_t)(m + 1));
  double* rd = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* b = (double*)malloc(sizeof(double) * (size_t)(m + 1));
  oracle_matvec(lp, x, ax);
  for (int i = 0; i < m; ++i) {
    const double rl = lp->row_lower[i], ru = lp->row_upper[i];
    if (rl == ru && is_fin(rl))
      rp[i] = rl - ax[i];
    else if (ax[i] < rl)
      rp[i] = rl - ax[i];
    else if (ax[i] > ru)
      rp[i] = ax[i] - ru;
    else
      rp[i] = 0.0;
  }
  double bv_inf = 0.0;
  for (int j = 0; j < n; ++j) {
    const double bv = max3(lp->col_lower[j] - x[j], x[j] - lp->col_upper[j], 0.0);
    bv_inf = j == 0 ? fabs(bv) : smax(bv_inf, fabs(bv));
  }
  oracle_matvec_transpose(lp, y, rd);
  for (int j = 0; j < n; ++j) rd[j] = rd[j] + z[j] - lp->c[j];
  rep->rp_norm2 = oracle_norm(rp, m);
  rep->rd_norm2 = oracle_norm(rd, n);
  double rp_inf = 0.0;
  for (int i = 0; i < m; ++i) rp_inf = i == 0 ? fabs(rp[i]) : smax(rp_inf, fabs(rp[i]));
  rep->rp_inf = smax(rp_inf, n ? bv_inf : 0.0);
  double rd_inf = 0.0;
  for (int j = 0; j < n; ++j) rd_inf = j == 0 ? fabs(rd[j]) : smax(rd_inf, fabs(rd[j]));
  rep->rd_inf = n ? rd_inf : 0.0;
  representative_rhs(lp, b);
  const double pobj = oracle_dot(lp->c, x, n);
  double dobj = oracle_dot(b, y, m);
  for (int j = 0; j < n; ++j) {
    const double zj = z[j];
    if (zj > 0.0 && is_fin(lp->col_lower[j]))
      dobj += lp->col_lower[j] * zj;
    else if (zj < 0.0 && is_fin(lp->col_upper[j]))
      dobj += lp->col_upper[j] * zj;
  }
  rep->primal_objective = pobj;
  rep->dual_objective = dobj;
  rep->gap_abs = fabs(pobj - dobj);
  rep->rel_primal = rep->rp_norm2 / (1.0 + oracle_norm(b, m));
  rep->rel_dual = rep->rd_norm2 / (1.0 + oracle_norm(lp->c, n));
  rep->rel_gap = rep->gap_abs / (1.0 + fabs(pobj) + fabs(dobj));
  rep->maxresid_rel = max3(rep->rel_primal, rep->rel_dual, rep->rel_gap);
  double worst = 0.0;
  for (int j = 0; j < n; ++j) {
    double dist = INFINITY;
    if (is_fin(lp->col_lower[j])) dist = smin(dist, fabs(x[j] - lp->col_lower[j]));
    if (is_fin(lp->col_upper[j])) dist = smin(dist, fabs(x[j] - lp->col_upper[j]));
    if (!is_fin(dist)) continue;
    worst = smax(worst, dist * fabs(z[j]));
  }
  rep->complementarity = worst;
  free(ax);
  free(rp);
  free(rd);
  free(b);
}

/* ---- run_pdhg (pdhg.cpp:230-378) --------------------------------------- */

typedef struct {
  double *x, *y, *z, *ax, *aty;
  oracle_report report;
} view_t;

typedef struct {
  const oracle_lp* lp;  /* unscaled std LP */
  const oracle_lp* slp; /* scaled */
  const double *r, *s;
  double b_norm, c_norm;
} ctx_t;

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* view_of (pdhg.cpp:271-283) + UnscaledView (:222-226). */
static void view_of(const ctx_t* c, const double* xs, const double* ys, const double* axs,
                    const double* atys, view_t* v) {
  const int m = c->lp->m, n = c->lp->n;
  for (int j = 0; j < n; ++j) v->x[j] = xs[j] * c->s[j];       /* unscale_x, scaling.hpp:31-33 */
  for (int i = 0; i < m; ++i) v->y[i] = ys[i] * c->r[i];       /* unscale_y, :34-36 */
  for (int i = 0; i < m; ++i) v->ax[i] = axs[i] / c->r[i];     /* pdhg.cpp:276 */
  for (int j = 0; j < n; ++j) v->aty[j] = atys[j] / c->s[j];   /* pdhg.cpp:277 */
  clipped_z(c->lp, v->x, v->aty, v->z);
  report_from_products(c->lp, v->x, v->y, v->z, v->ax, v->aty, c->b_norm, c->c_norm, &v->report);
}

static void view_alloc(view_t* v, int m, int n) {
  v->x = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  v->z = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  v->aty = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  v->y = (double*)malloc(sizeof(double) * (size_t)(m + 1));
  v->ax = (double*)malloc(sizeof(double) * (size_t)(m + 1));
}
static void view_free(view_t* v) {
  free(v->x);
  free(v->z);
  free(v->aty);
  free(v->y);
  free(v->ax);
}

static int all_finite(const double* a, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (isnan(a[i] - a[i])) return 0;
  return 1;
}

int oracle_run_pdhg(const oracle_lp* lp, const oracle_config* cfg, const oracle_tol* tol,
                    const double* thresholds, int nthr, oracle_sink sink, void* sink_user,
                    const volatile uint8_t* cancel, double* x_out, double* y_out, double* z_out,
                    oracle_result* res, oracle_trace* trace) {
  const int m = lp->m, n = lp->n;
  /* Preconditions (pdhg.cpp:235-244, kkt.cpp:26-37). */
  for (int i = 0; i < m; ++i) {
    if (!(lp->row_lower[i] == lp->row_upper[i] && is_fin(lp->row_lower[i]))) {
      snprintf(g_err, sizeof g_err, "run_pdhg: LP must be in equality form");
      return 1;
    }
  }
  if (!(tol->decrement > 0.0 && tol->decrement < 1.0)) {
    snprintf(g_err, sizeof g_err, "tolerances: decrement must be in (0,1)");
    return 1;
  }
  if (!(tol->eps_rel > 0.0 && tol->eps_rel <= tol->eps_cross)) {
    snprintf(g_err, sizeof g_err, "tolerances: need 0 < eps_rel <= eps_cross");
    return 1;
  }
  if (!(tol->eps_abs > 0.0)) {
    snprintf(g_err, sizeof g_err, "tolerances: eps_abs must be positive");
    return 1;
  }
  for (int i = 1; i < nthr; ++i) {
    if (!(thresholds[i] < thresholds[i - 1])) {
      snprintf(g_err, sizeof g_err, "run_pdhg: thresholds must be strictly decreasing");
      return 1;
    }
  }
  if (cfg->check_interval <= 0) { /* modulo by zero in the reference (pdhg.cpp:311) */
    snprintf(g_err, sizeof g_err, "run_pdhg: check_interval must be positive");
    return 1;
  }
  const double t0 = now_s();
  const int nnz = lp->colptr[n];

  /* ruiz_scale (pdhg.cpp:252). */
  double* r = (double*)malloc(sizeof(double) * (size_t)(m + 1));
  double* s = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* sval = (double*)malloc(sizeof(double) * (size_t)(nnz + 1));
  oracle_ruiz(lp, cfg->scaling_iterations, r, s, sval);
  double* sc = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* sl = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* su = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* sb = (double*)malloc(sizeof(double) * (size_t)(m + 1));
  for (int j = 0; j < n; ++j) {
    sc[j] = lp->c[j] * s[j];
    sl[j] = lp->col_lower[j] / s[j];
    su[j] = lp->col_upper[j] / s[j];
  }
  for (int i = 0; i < m; ++i) sb[i] = lp->row_lower[i] * r[i];
  oracle_lp slp = {m, n, lp->colptr, lp->rowind, sval, sc, sb, sb, sl, su};

  double* tmpb = (double*)malloc(sizeof(double) * (size_t)(m + 1));
  representative_rhs(lp, tmpb);
  ctx_t cx = {lp, &slp, r, s, oracle_norm(tmpb, m), oracle_norm(lp->c, n)}; /* :253-254 */

  /* make_initial_state (pdhg.cpp:67-82) on the scaled LP. */
  double* x = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* aty = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* x_sum = (double*)calloc((size_t)(n + 1), sizeof(double));
  double* aty_sum = (double*)calloc((size_t)(n + 1), sizeof(double));
  double* y = (double*)calloc((size_t)(m + 1), sizeof(double));
  double* ax = (double*)malloc(sizeof(double) * (size_t)(m + 1));
  double* y_sum = (double*)calloc((size_t)(m + 1), sizeof(double));
  double* ax_sum = (double*)calloc((size_t)(m + 1), sizeof(double));
  double* xn = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* atyn = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* yn = (double*)malloc(sizeof(double) * (size_t)(m + 1));
  double* axn = (double*)malloc(sizeof(double) * (size_t)(m + 1));
  double* xa = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* atya = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* ya = (double*)malloc(sizeof(double) * (size_t)(m + 1));
  double* axa = (double*)malloc(sizeof(double) * (size_t)(m + 1));
  for (int j = 0; j < n; ++j) x[j] = smin(smax(0.0, sl[j]), su[j]); /* Zero.cwiseMax(l).cwiseMin(u) */
  oracle_matvec(&slp, x, ax);
  oracle_matvec_transpose(&slp, y, aty);

  /* ||A|| and step sizes (pdhg.cpp:257-267). */
  const double norm_est = oracle_estimate_norm(&slp, cfg->norm_iterations, cfg->seed);
  const double a_norm = norm_est > 0.0 ? norm_est : 1.0;
  double omega = cfg->primal_weight;
  if (omega <= 0.0) {
    representative_rhs(&slp, tmpb);
    const double cs = oracle_norm(sc, n), bs = oracle_norm(tmpb, m);
    omega = (cs > 0.0 && bs > 0.0) ? cs / bs : 1.0;
  }
  const double tau = cfg->step_scale * omega / a_norm;
  const double sigma = cfg->step_scale / (omega * a_norm);

  int64_t window = 0, iteration = 0, restarts = 0;
  double last_restart_resid = INFINITY;
  int next_threshold = 0;
  int have_best = 0;
  oracle_report best;
  memset(&best, 0, sizeof best);
  view_t cur, avg, fin;
  view_alloc(&cur, m, n);
  view_alloc(&avg, m, n);
  view_alloc(&fin, m, n);
  int stop = -1;
  view_t* out_view = &fin;
  int64_t error_iteration = -1;

  while (1) {
    if (cancel != NULL && *cancel) { /* :301-305 */
      stop = ORACLE_CANCELLED;
      view_of(&cx, x, y, ax, aty, &fin);
      break;
    }
    if (now_s() - t0 > cfg->time_limit) { /* :306-310 */
      stop = ORACLE_TIME_LIMIT;
      view_of(&cx, x, y, ax, aty, &fin);
      break;
    }
    if (iteration % cfg->check_interval == 0) { /* :311-363 */
      view_of(&cx, x, y, ax, aty, &cur);
      int use_avg = 0;
      if (window > 0) {
        const double inv = 1.0 / (double)window;
        for (int j = 0; j < n; ++j) xa[j] = x_sum[j] * inv;
        for (int i = 0; i < m; ++i) ya[i] = y_sum[i] * inv;
        for (int i = 0; i < m; ++i) axa[i] = ax_sum[i] * inv;
        for (int j = 0; j < n; ++j) atya[j] = aty_sum[j] * inv;
        view_of(&cx, xa, ya, axa, atya, &avg);
        use_avg = avg.report.maxresid_rel < cur.report.maxresid_rel;
      }
      view_t* better = use_avg ? &avg : &cur;
      if (!have_best || better->report.maxresid_rel < best.maxresid_rel) {
        best = better->report;
        have_best = 1;
      }
      if (last_restart_resid == INFINITY) last_restart_resid = cur.report.maxresid_rel;
      if (trace && trace->trace && trace->n_trace < trace->trace_cap) {
        trace->trace[3 * trace->n_trace + 0] = (double)iteration;
        trace->trace[3 * trace->n_trace + 1] = cur.report.maxresid_rel;
        trace->trace[3 * trace->n_trace + 2] = window > 0 ? avg.report.maxresid_rel : -1.0;
        trace->n_trace++;
      }
      if (better->report.maxresid_rel <= tol->eps_rel) {
        stop = ORACLE_CONVERGED;
        out_view = better;
        break;
      }
      if (next_threshold < nthr && better->report.maxresid_rel <= thresholds[next_threshold]) {
        if (sink) {
          oracle_snapshot snap = {thresholds[next_threshold], better->report.maxresid_rel, use_avg,
                                  iteration, better->x, better->y, better->z};
          sink(&snap, sink_user);
        }
        ++next_threshold;
      }
      if (window > 0) { /* restart_if_improved (pdhg.cpp:145-165) */
        if (window >= 1 && avg.report.maxresid_rel <= cfg->restart_factor * last_restart_resid) {
          const double inv = 1.0 / (double)window;
          for (int j = 0; j < n; ++j) x[j] = x_sum[j] * inv;
          for (int i = 0; i < m; ++i) y[i] = y_sum[i] * inv;
          for (int i = 0; i < m; ++i) ax[i] = ax_sum[i] * inv;
          for (int j = 0; j < n; ++j) aty[j] = aty_sum[j] * inv;
          memset(x_sum, 0, sizeof(double) * (size_t)n);
          memset(y_sum, 0, sizeof(double) * (size_t)m);
          memset(ax_sum, 0, sizeof(double) * (size_t)m);
          memset(aty_sum, 0, sizeof(double) * (size_t)n);
          window = 0;
          last_restart_resid = avg.report.maxresid_rel;
          ++restarts;
          if (trace && trace->restart_iters && trace->n_restarts_logged < trace->restart_cap)
            trace->restart_iters[trace->n_restarts_logged++] = iteration;
        }
      }
    }
    if (iteration >= cfg->max_iterations) { /* :364-368 */
      stop = ORACLE_ITERATION_LIMIT;
      view_of(&cx, x, y, ax, aty, &fin);
      break;
    }
    /* pdhg_step (pdhg.cpp:118-143). */
    for (int j = 0; j < n; ++j) {
      double t = sc[j] - aty[j];
      t = tau * t;
      t = x[j] - t;
      t = smax(t, sl[j]); /* cwiseMax: (t < l) ? l : t */
      xn[j] = smin(t, su[j]);
    }
    oracle_matvec(&slp, xn, axn);
    for (int i = 0; i < m; ++i) {
      double t = 2.0 * axn[i];
      t = t - ax[i];
      t = sb[i] - t;
      t = sigma * t;
      yn[i] = y[i] + t;
    }
    oracle_matvec_transpose(&slp, yn, atyn);
    if (!all_finite(xn, n) || !all_finite(yn, m)) { /* :128-130, :369-376 */
      error_iteration = iteration;
      stop = ORACLE_NUMERICAL_ERROR;
      view_of(&cx, x, y, ax, aty, &fin);
      break;
    }
    double* t;
    t = x; x = xn; xn = t;
    t = y; y = yn; yn = t;
    t = ax; ax = axn; axn = t;
    t = aty; aty = atyn; atyn = t;
    ++iteration;
    for (int j = 0; j < n; ++j) x_sum[j] = x_sum[j] + x[j];
    for (int i = 0; i < m; ++i) y_sum[i] = y_sum[i] + y[i];
    for (int i = 0; i < m; ++i) ax_sum[i] = ax_sum[i] + ax[i];
    for (int j = 0; j < n; ++j) aty_sum[j] = aty_sum[j] + aty[j];
    ++window;
  }

  memcpy(x_out, out_view->x, sizeof(double) * (size_t)n);
  memcpy(y_out, out_view->y, sizeof(double) * (size_t)m);
  memcpy(z_out, out_view->z, sizeof(double) * (size_t)n);
  res->stop = stop;
  res->report = out_view->report;
  res->iterations = iteration;
  res->restarts = restarts;
  res->error_iteration = error_iteration;
  res->seconds = now_s() - t0;
  res->tau = tau;
  res->sigma = sigma;
  res->norm_estimate = norm_est;
  res->omega = omega;

  view_free(&cur);
  view_free(&avg);
  view_free(&fin);
  free(r); free(s); free(sval); free(sc); free(sl); free(su); free(sb); free(tmpb);
  free(x); free(aty); free(x_sum); free(aty_sum); free(y); free(ax); free(y_sum); free(ax_sum);
  free(xn); free(atyn); free(yn); free(axn); free(xa); free(atya); free(ya); free(axa);
  return 0;
}
