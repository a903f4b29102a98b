// C-ABI bridge to the REFERENCE implementation — TEST INFRASTRUCTURE ONLY.
//
// Compiled together with the reference's own, unmodified sources
// (/root/reference/proj/src/{lp,kernels,scaling,kkt,pdhg,standard_form}.cpp)
// into oracle/_ref/libcclp_ref.so, so that Python tests, the golden-fixture
// generator and bench.py's reference arm can call the genuine
// cclp::run_pdhg (pdhg.hpp:138-142) and its helpers through ctypes.
// Only tests/, __graft_entry__.smoke() and bench.py's CPU legs load it.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "cclp/kernels.hpp"
#include "cclp/kkt.hpp"
#include "cclp/lp.hpp"
#include "cclp/pdhg.hpp"
#include "cclp/scaling.hpp"

namespace {

thread_local std::string g_err;

cclp::Vector vec(const double* p, int n) {
  cclp::Vector v(n);
  if (n > 0) std::memcpy(v.data(), p, sizeof(double) * static_cast<size_t>(n));
  return v;
}

void put(const cclp::Vector& v, double* out) {
  if (out != nullptr && v.size() > 0)
    std::memcpy(out, v.data(), sizeof(double) * static_cast<size_t>(v.size()));
}

cclp::SparseMat csc(int m, int n, const int* colptr, const int* rowind, const double* val) {
  return cclp::SparseMat(Eigen::Map<cclp::SparseMat>(m, n, colptr[n], colptr, rowind, val));
}

cclp::LinearProgram make_lp(int m, int n, const int* colptr, const int* rowind, const double* val,
                            const double* c, const double* rl, const double* ru, const double* cl,
                            const double* cu) {
  cclp::LinearProgram lp;
  lp.A = csc(m, n, colptr, rowind, val);
  lp.c = vec(c, n);
  lp.row_lower = vec(rl, m);
  lp.row_upper = vec(ru, m);
  lp.col_lower = vec(cl, n);
  lp.col_upper = vec(cu, n);
  lp.sense.assign(static_cast<size_t>(m), cclp::RowSense::kEq);
  for (int i = 0; i < m; ++i) {
    if (rl[i] != ru[i]) lp.sense[static_cast<size_t>(i)] = cclp::RowSense::kLe;
  }
  return lp;
}

void put_report(const cclp::ResidualReport& r, double* out) {
  if (out == nullptr) return;
  const double v[12] = {r.rp_norm2,         r.rd_norm2,       r.rp_inf,  r.rd_inf,
                        r.primal_objective, r.dual_objective, r.gap_abs, r.rel_primal,
                        r.rel_dual,         r.rel_gap,        r.maxresid_rel, r.complementarity};
  std::memcpy(out, v, sizeof v);
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // namespace

extern "C" {

const char* cclp_ref_last_error(void) { return g_err.c_str(); }

int cclp_ref_matvec(int m, int n, const int* colptr, const int* rowind, const double* val,
                    const double* x, double* out) {
  return guarded([&] { put(cclp::matvec(csc(m, n, colptr, rowind, val), vec(x, n)), out); });
}

int cclp_ref_matvec_transpose(int m, int n, const int* colptr, const int* rowind, const double* val,
                              const double* y, double* out) {
  return guarded(
      [&] { put(cclp::matvec_transpose(csc(m, n, colptr, rowind, val), vec(y, m)), out); });
}

int cclp_ref_estimate_norm(int m, int n, const int* colptr, const int* rowind, const double* val,
                           int iterations, uint64_t seed, double* out) {
  return guarded([&] {
    *out = cclp::estimate_matrix_norm(csc(m, n, colptr, rowind, val), iterations, seed);
  });
}

// Ruiz factors plus the scaled matrix values / objective / bounds.
int cclp_ref_ruiz(int m, int n, const int* colptr, const int* rowind, const double* val,
                  const double* c, const double* rl, const double* ru, const double* cl,
                  const double* cu, int iterations, double* row_scale, double* col_scale,
                  double* scaled_val, double* scaled_c, double* scaled_b) {
  return guarded([&] {
    auto lp = make_lp(m, n, colptr, rowind, val, c, rl, ru, cl, cu);
    auto [slp, info] = cclp::ruiz_scale(lp, iterations);
    put(info.row_scale, row_scale);
    put(info.col_scale, col_scale);
    if (scaled_val != nullptr && slp.A.nonZeros() > 0)
      std::memcpy(scaled_val, slp.A.valuePtr(), sizeof(double) * static_cast<size_t>(slp.A.nonZeros()));
    put(slp.c, scaled_c);
    put(slp.row_lower, scaled_b);
  });
}

int cclp_ref_relative_report(int m, int n, const int* colptr, const int* rowind, const double* val,
                             const double* c, const double* rl, const double* ru, const double* cl,
                             const double* cu, const double* x, const double* y, const double* z,
                             double* report) {
  return guarded([&] {
    auto lp = make_lp(m, n, colptr, rowind, val, c, rl, ru, cl, cu);
    cclp::Iterate it;
    it.x = vec(x, n);
    it.y = vec(y, m);
    it.z = vec(z, n);
    put_report(cclp::relative_report(lp, it), report);
  });
}

// dcfg: step_scale, primal_weight, restart_factor, time_limit
// icfg: norm_iterations, scaling_iterations, max_iterations, check_interval, seed
// tol : eps_rel, eps_abs, eps_cross, decrement
// stats_out: stop, iterations, restarts, error_iteration
// snap_meta (4 per snapshot): threshold, maxresid, from_average, iteration
int cclp_ref_run_pdhg(int m, int n, const int* colptr, const int* rowind, const double* val,
                      const double* c, const double* rl, const double* ru, const double* cl,
                      const double* cu, const double* dcfg, const int64_t* icfg, const double* tol,
                      const double* thresholds, int nthr, const uint8_t* cancel_flag,
                      double* x_out, double* y_out, double* z_out, double* report_out,
                      int64_t* stats_out, double* seconds_out, double* snap_x, double* snap_y,
                      double* snap_z, double* snap_meta, int* nsnap) {
  return guarded([&] {
    auto lp = make_lp(m, n, colptr, rowind, val, c, rl, ru, cl, cu);
    cclp::PdhgConfig cfg;
    cfg.step_scale = dcfg[0];
    cfg.primal_weight = dcfg[1];
    cfg.restart_factor = dcfg[2];
    cfg.time_limit = dcfg[3];
    cfg.norm_iterations = static_cast<int>(icfg[0]);
    cfg.scaling_iterations = static_cast<int>(icfg[1]);
    cfg.max_iterations = icfg[2];
    cfg.check_interval = static_cast<int>(icfg[3]);
    cfg.seed = static_cast<uint64_t>(icfg[4]);
    cclp::Tolerances t;
    t.eps_rel = tol[0];
    t.eps_abs = tol[1];
    t.eps_cross = tol[2];
    t.decrement = tol[3];
    std::vector<double> thr(thresholds, thresholds + nthr);
    int count = 0;
    auto sink = [&](const cclp::PdhgSnapshot& s) {
      if (snap_x != nullptr) put(s.iterate.x, snap_x + static_cast<size_t>(count) * n);
      if (snap_y != nullptr) put(s.iterate.y, snap_y + static_cast<size_t>(count) * m);
      if (snap_z != nullptr) put(s.iterate.z, snap_z + static_cast<size_t>(count) * n);
      if (snap_meta != nullptr) {
        snap_meta[4 * count + 0] = s.threshold;
        snap_meta[4 * count + 1] = s.maxresid;
        snap_meta[4 * count + 2] = s.from_average ? 1.0 : 0.0;
        snap_meta[4 * count + 3] = static_cast<double>(s.iteration);
      }
      ++count;
    };
    std::atomic<bool> cancel{cancel_flag != nullptr && *cancel_flag != 0};
    cclp::PdhgResult r = cclp::run_pdhg(lp, cfg, t, thr, sink, &cancel);
    put(r.iterate.x, x_out);
    put(r.iterate.y, y_out);
    put(r.iterate.z, z_out);
    put_report(r.report, report_out);
    stats_out[0] = static_cast<int64_t>(r.stop);
    stats_out[1] = r.iterations;
    stats_out[2] = r.restarts;
    stats_out[3] = r.error_iteration;
    if (seconds_out != nullptr) *seconds_out = r.seconds;
    if (nsnap != nullptr) *nsnap = count;
  });
}

}  // extern "C"
