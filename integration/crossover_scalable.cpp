// Scalable crossover (crossover_scalable.hpp): the reference's run_crossover
// algorithm (crossover.cpp:247-285, simplex.cpp:119-426) over sparse basis
// factors and device pricing. Every step cites the reference line it
// restates; the numerical kernels (sparse LU, sparse etas) are this repo's.
#include "crossover_scalable.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "cclp/basis.hpp"
#include "cclp/kkt.hpp"
#include "cclp/simplex.hpp"
#ifndef CCLP_XO_NO_DEVICE
#include "cclp_cu.h"
#endif

namespace cclp_xo {

using cclp::Basis;
using cclp::ColStatus;
using cclp::EngineModel;
using cclp::Index;
using cclp::LinearProgram;
using cclp::Scalar;
using cclp::Vector;
using Clock = std::chrono::steady_clock;

// ---------------------------------------------------------------------------
// Device pricer
// ---------------------------------------------------------------------------
#ifndef CCLP_XO_NO_DEVICE
DevicePricer::DevicePricer(const LinearProgram& lp, int device) {
  cclp_cu_lp d{};
  d.m = lp.num_rows();
  d.n = lp.num_cols();
  d.colptr = lp.A.outerIndexPtr();
  d.rowind = lp.A.innerIndexPtr();
  d.val = lp.A.valuePtr();
  d.c = lp.c.data();
  d.row_lower = lp.row_lower.data();
  d.row_upper = lp.row_upper.data();
  d.col_lower = lp.col_lower.data();
  d.col_upper = lp.col_upper.data();
  if (cclp_cu_create(&d, device, &ctx_) != CCLP_CU_OK)
    throw std::runtime_error(std::string("DevicePricer: ") + cclp_cu_last_error());
}
DevicePricer::~DevicePricer() {
  if (ctx_) cclp_cu_destroy(ctx_);
}
void DevicePricer::price(const double* y, const char* status, const unsigned char* skip, bool phase1, double dtol,
                         bool bland, long long* entering, int* direction, double* violation) {
  std::lock_guard<std::mutex> g(mu_);
  int64_t e = -1;
  int32_t d = 0;
  if (cclp_cu_price(ctx_, y, status, skip, phase1 ? 1 : 0, dtol, bland ? 1 : 0, &e, &d, violation) != CCLP_CU_OK)
    throw std::runtime_error(std::string("DevicePricer: ") + cclp_cu_last_error());
  *entering = e;
  *direction = d;
  ++calls_;
}
#else
DevicePricer::DevicePricer(const LinearProgram&, int) {
  throw std::runtime_error("DevicePricer: built without the B200 engine");
}
DevicePricer::~DevicePricer() = default;
void DevicePricer::price(const double*, const char*, const unsigned char*, bool, double, bool, long long*, int*,
                         double*) {}
#endif

namespace {

// Engine column j of [A | I] (basis.hpp:33-47): structural from the CSC,
// logical n + i = e_i.
struct Cols {
  const int* ptr;
  const int* idx;
  const double* val;
  int n;
  int len(Index j) const { return j < n ? ptr[j + 1] - ptr[j] : 1; }
  template <class F>
  void each(Index j, F&& f) const {
    if (j >= n) {
      f(static_cast<int>(j - n), 1.0);
      return;
    }
    for (int p = ptr[j]; p < ptr[j + 1]; ++p) f(idx[p], val[p]);
  }
};

Cols cols_of(const LinearProgram& lp) {
  return Cols{lp.A.outerIndexPtr(), lp.A.innerIndexPtr(), lp.A.valuePtr(), static_cast<int>(lp.num_cols())};
}

// Depth-first reach of `starts` in the graph "node v -> targets of column
// col_of(v)" (Gilbert-Peierls): nodes in reverse topological order.
template <class ColOf, class Adj>
void reach(const std::vector<int>& starts, std::vector<int>& mark, int stamp, ColOf col_of, Adj adj,
           std::vector<int>& out, std::vector<int>& stack, std::vector<int>& pos) {
  out.clear();
  for (int s : starts) {
    if (mark[s] == stamp) continue;
    mark[s] = stamp;
    stack.assign(1, s);
    pos.assign(1, 0);
    while (!stack.empty()) {
      const int v = stack.back();
      const int c = col_of(v);
      bool pushed = false;
      if (c >= 0) {
        int& k = pos.back();
        const int* b;
        const int* e;
        adj(c, b, e);
        for (const int* t = b + k; t < e; ++t) {
          ++k;
          const int w = *t;
          if (mark[w] == stamp) continue;
          mark[w] = stamp;
          stack.push_back(w);
          pos.push_back(0);
          pushed = true;
          break;
        }
      }
      if (!pushed) {
        out.push_back(v);
        stack.pop_back();
        pos.pop_back();
      }
    }
  }
}

// ---------------------------------------------------------------------------
// The crash (build_basis, crossover.cpp:101-150) as an incremental
// left-looking LU over the identity: accepted candidate k pivots on row
// piv[k]; for a new column a, x = L^{-1} a holds at unpivoted rows the
// entries of w = B^{-1} a at the still-logical positions and at pivoted rows
// the right-hand side of U z = x_piv, z = w at the accepted positions.
// ---------------------------------------------------------------------------
class CrashLU {
 public:
  explicit CrashLU(int m) : m_(m), pinv_(m, -1), mark_(m, -1), smark_(1, -1), x_(m, 0.0) {
    lp_.push_back(0);
    up_.push_back(0);
  }

  // One candidate; returns the pivot row (= the replaced position) or -1.
  int offer(const Cols& cols, Index j) {
    ++stamp_;
    starts_.clear();
    cols.each(j, [&](int r, double v) {
      starts_.push_back(r);
      x_[r] = v;
    });
    // pattern of L^{-1} a: through the L columns of pivoted rows
    reach(
        starts_, mark_, stamp_, [&](int r) { return pinv_[r]; },
        [&](int c, const int*& b, const int*& e) {
          b = li_.data() + lp_[c] + 1;  // skip the unit diagonal
          e = li_.data() + lp_[c + 1];
        },
        topo_, stack_, pos_);
    for (auto it = topo_.rbegin(); it != topo_.rend(); ++it) {
      const int r = *it;
      const int c = pinv_[r];
      if (c < 0) continue;
      const double xr = x_[r];
      if (xr == 0.0) continue;
      for (int t = lp_[c] + 1; t < lp_[c + 1]; ++t) x_[li_[t]] = x_[li_[t]] - lx_[t] * xr;
    }
    // w at the still-logical positions; the pivot: largest, lowest row on ties
    int best = -1;
    double best_abs = 0.0, wmax = 0.0;
    piv_steps_.clear();
    for (int r : topo_) {
      const double mag = std::abs(x_[r]);
      if (pinv_[r] >= 0) {
        piv_steps_.push_back(pinv_[r]);
        continue;
      }
      wmax = std::max(wmax, mag);
      if (mag > best_abs || (mag == best_abs && mag > 0.0 && r < best)) {
        best_abs = mag;
        best = r;
      }
    }
    // w at the accepted positions: z = U^{-1} x_piv (only for ||w||_inf)
    if (!piv_steps_.empty()) {
      const int k = static_cast<int>(up_.size()) - 1;
      if (static_cast<int>(z_.size()) < k) {
        z_.resize(k, 0.0);
        smark_.resize(k, -1);
      }
      for (int r : topo_)
        if (pinv_[r] >= 0) z_[pinv_[r]] = x_[r];
      reach(
          piv_steps_, smark_, stamp_, [](int s) { return s; },
          [&](int s, const int*& b, const int*& e) {
            b = ui_.data() + up_[s];
            e = ui_.data() + up_[s + 1] - 1;  // the diagonal is last
          },
          ztopo_, stack_, pos_);
      for (auto it = ztopo_.rbegin(); it != ztopo_.rend(); ++it) {
        const int s = *it;
        const int dpos = up_[s + 1] - 1;
        const double zs = z_[s] / ux_[dpos];
        z_[s] = zs;
        wmax = std::max(wmax, std::abs(zs));
        if (zs == 0.0) continue;
        for (int t = up_[s]; t < dpos; ++t) z_[ui_[t]] = z_[ui_[t]] - ux_[t] * zs;
      }
      for (int s : ztopo_) z_[s] = 0.0;
    }
    // dependent on the accepted set (or numerically too risky): skip (:131-133)
    const bool take = best >= 0 && !(best_abs < 1e-7 * std::max(1.0, wmax));
    if (take) {
      const int k = static_cast<int>(up_.size()) - 1;
      const double d = x_[best];
      for (int r : topo_)
        if (pinv_[r] >= 0 && x_[r] != 0.0) {
          ui_.push_back(pinv_[r]);
          ux_.push_back(x_[r]);
        }
      ui_.push_back(k);
      ux_.push_back(d);
      up_.push_back(static_cast<int>(ui_.size()));
      pinv_[best] = k;
      li_.push_back(best);
      lx_.push_back(1.0);
      for (int r : topo_)
        if (pinv_[r] < 0 && x_[r] != 0.0) {
          li_.push_back(r);
          lx_.push_back(x_[r] / d);
        }
      lp_.push_back(static_cast<int>(li_.size()));
    }
    for (int r : topo_) x_[r] = 0.0;
    return take ? best : -1;
  }
  long long nnz() const { return static_cast<long long>(li_.size() + ui_.size()); }

 private:
  int m_;
  std::vector<int> pinv_, mark_, smark_;
  std::vector<double> x_, z_;
  std::vector<int> lp_, li_, up_, ui_;
  std::vector<double> lx_, ux_;
  std::vector<int> starts_, topo_, ztopo_, piv_steps_, stack_, pos_;
  int stamp_ = 0;
};

// ---------------------------------------------------------------------------
// Basis factorization for the simplex (FactorizedBasis, factorization.cpp:
// 58-139): P B Q = L U, sparse left-looking with threshold partial pivoting
// (Markowitz-style row choice) and columns by increasing length; rank-
// revealing (a column without a pivot above 1e-10 max(1, max|B|), the
// dependent_positions tolerance, is reported and skipped). Product-form
// updates keep SPARSE eta vectors.
// ---------------------------------------------------------------------------
class SparseBasis {
 public:
  SparseBasis(const Cols& cols, int m) : cols_(cols), m_(m) {}

  // false: the positions without a pivot in `dependent` (ascending) and the
  // rows left unpivoted in `free_rows` (ascending).
  bool factorize(const std::vector<Index>& basic, std::vector<Index>* dependent, std::vector<int>* free_rows) {
    const int m = m_;
    etas_.clear();
    q_.assign(m, -1);
    pinv_.assign(m, -1);
    lp_.assign(1, 0);
    up_.assign(1, 0);
    li_.clear(); lx_.clear(); ui_.clear(); ux_.clear();
    std::vector<int> rowcnt(m, 0);
    double scale = 1.0;
    for (int k = 0; k < m; ++k)
      cols_.each(basic[k], [&](int r, double v) {
        ++rowcnt[r];
        scale = std::max(scale, std::abs(v));
      });
    const double tol = 1e-10 * scale;
    std::vector<int> order(m);
    for (int k = 0; k < m; ++k) order[k] = k;
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return cols_.len(basic[a]) < cols_.len(basic[b]); });
    std::vector<double> x(m, 0.0);
    std::vector<int> mark(m, -1), starts, topo, stack, pos;
    dependent->clear();
    int step = 0;
    for (int t = 0; t < m; ++t) {
      const int k = order[t];
      starts.clear();
      cols_.each(basic[k], [&](int r, double v) {
        starts.push_back(r);
        x[r] = v;
      });
      reach(
          starts, mark, t, [&](int r) { return pinv_[r]; },
          [&](int c, const int*& b, const int*& e) {
            b = li_.data() + lp_[c] + 1;
            e = li_.data() + lp_[c + 1];
          },
          topo, stack, pos);
      for (auto it = topo.rbegin(); it != topo.rend(); ++it) {
        const int r = *it;
        const int c = pinv_[r];
        if (c < 0) continue;
        const double xr = x[r];
        if (xr == 0.0) continue;
        for (int u = lp_[c] + 1; u < lp_[c + 1]; ++u) x[li_[u]] = x[li_[u]] - lx_[u] * xr;
      }
      double colmax = 0.0;
      for (int r : topo)
        if (pinv_[r] < 0) colmax = std::max(colmax, std::abs(x[r]));
      if (!(colmax > tol)) {
        dependent->push_back(k);
        for (int r : topo) x[r] = 0.0;
        continue;
      }
      int piv = -1;
      double pv = 0.0;
      for (int r : topo) {
        if (pinv_[r] >= 0) continue;
        const double v = std::abs(x[r]);
        if (v < 0.1 * colmax) continue;
        if (piv < 0 || rowcnt[r] < rowcnt[piv] || (rowcnt[r] == rowcnt[piv] && (v > pv || (v == pv && r < piv)))) {
          piv = r;
          pv = v;
        }
      }
      const double d = x[piv];
      for (int r : topo)
        if (pinv_[r] >= 0 && x[r] != 0.0) {
          ui_.push_back(pinv_[r]);
          ux_.push_back(x[r]);
        }
      ui_.push_back(step);
      ux_.push_back(d);
      up_.push_back(static_cast<int>(ui_.size()));
      pinv_[piv] = step;
      li_.push_back(piv);
      lx_.push_back(1.0);
      for (int r : topo) {
        if (pinv_[r] < 0 && x[r] != 0.0) {
          li_.push_back(r);
          lx_.push_back(x[r] / d);
        }
        x[r] = 0.0;
      }
      lp_.push_back(static_cast<int>(li_.size()));
      q_[step] = k;
      ++step;
    }
    if (!dependent->empty()) {
      std::sort(dependent->begin(), dependent->end());
      free_rows->clear();
      for (int r = 0; r < m; ++r)
        if (pinv_[r] < 0) free_rows->push_back(r);
      return false;
    }
    for (int& r : li_) r = pinv_[r];  // rows of L by step from here on
    return true;
  }

  // x (by rows) -> B^{-1} x (by positions), etas applied (factorization.cpp:106-115)
  void ftran(std::vector<double>& x) const {
    const int m = m_;
    std::vector<double> w(m);
    for (int i = 0; i < m; ++i) w[pinv_[i]] = x[i];
    for (int k = 0; k < m; ++k) {
      const double wk = w[k];
      if (wk == 0.0) continue;
      for (int t = lp_[k] + 1; t < lp_[k + 1]; ++t) w[li_[t]] = w[li_[t]] - lx_[t] * wk;
    }
    for (int k = m - 1; k >= 0; --k) {
      const int dpos = up_[k + 1] - 1;
      const double wk = w[k] / ux_[dpos];
      w[k] = wk;
      if (wk == 0.0) continue;
      for (int t = up_[k]; t < dpos; ++t) w[ui_[t]] = w[ui_[t]] - ux_[t] * wk;
    }
    for (int k = 0; k < m; ++k) x[q_[k]] = w[k];
    for (const Eta& e : etas_) {
      const double t = x[e.p] / e.wp;
      if (t != 0.0)
        for (size_t q = 0; q < e.idx.size(); ++q) x[e.idx[q]] = x[e.idx[q]] - t * e.val[q];
      x[e.p] = t;
    }
  }
  // x (by positions) -> B^{-T} x (by rows) (factorization.cpp:117-125)
  void btran(std::vector<double>& x) const {
    const int m = m_;
    for (auto it = etas_.rbegin(); it != etas_.rend(); ++it) {
      const Eta& e = *it;
      double dot = 0.0;
      for (size_t q = 0; q < e.idx.size(); ++q)
        if (e.idx[q] != e.p) dot += e.val[q] * x[e.idx[q]];
      x[e.p] = (x[e.p] - dot) / e.wp;
    }
    std::vector<double> w(m);
    for (int k = 0; k < m; ++k) w[k] = x[q_[k]];
    for (int k = 0; k < m; ++k) {
      const int dpos = up_[k + 1] - 1;
      double s = w[k];
      for (int t = up_[k]; t < dpos; ++t) s = s - ux_[t] * w[ui_[t]];
      w[k] = s / ux_[dpos];
    }
    for (int k = m - 1; k >= 0; --k) {
      double s = w[k];
      for (int t = lp_[k] + 1; t < lp_[k + 1]; ++t) s = s - lx_[t] * w[li_[t]];
      w[k] = s;
    }
    for (int i = 0; i < m; ++i) x[i] = w[pinv_[i]];
  }
  // factorization.cpp:127-136, with w kept sparse
  void update(int slot, const std::vector<double>& w) {
    if (w[slot] == 0.0) throw cclp::SingularBasisError("basis update with zero pivot", {});
    Eta e;
    e.p = slot;
    e.wp = w[slot];
    for (int i = 0; i < m_; ++i)
      if (w[i] != 0.0) {
        e.idx.push_back(i);
        e.val.push_back(w[i]);
      }
    etas_.push_back(std::move(e));
  }
  int updates() const { return static_cast<int>(etas_.size()); }
  long long nnz() const { return static_cast<long long>(li_.size() + ui_.size()); }

 private:
  struct Eta {
    int p;
    double wp;
    std::vector<int> idx;
    std::vector<double> val;
  };
  Cols cols_;
  int m_;
  std::vector<int> q_, pinv_, lp_, li_, up_, ui_;
  std::vector<double> lx_, ux_;
  std::vector<Eta> etas_;
};

// ---------------------------------------------------------------------------
// Two-phase bounded primal simplex (simplex.cpp:119-426), restated over
// SparseBasis and a pricer.
// ---------------------------------------------------------------------------
constexpr Scalar kPivotTol = 1e-7;        // simplex.cpp:117
constexpr Scalar kDegenerateStep = 1e-11;  // simplex.cpp:118

class Simplex {
 public:
  Simplex(const LinearProgram& lp, const Basis& start, const cclp::SimplexOptions& opt, DevicePricer* pricer,
          ScalableStats* stats)
      : model_(lp), lp_(lp), cols_(cols_of(lp)), opt_(opt), basis_(start), pricer_(pricer), stats_(stats),
        factor_(cols_, lp.num_rows()), t0_(Clock::now()) {
    basis_.validate(model_);  // :123-134
    ftol_ = std::min(opt_.eps_abs, 1e-9);
    dtol_ = std::min(opt_.eps_abs, 1e-9);
    x_ = Vector::Zero(model_.num_cols());
    for (Index j = 0; j < model_.num_cols(); ++j)
      if (basis_.status[j] != ColStatus::kBasic) x_[j] = basis_.nonbasic_value(model_, j);
    status_.resize(model_.num_cols());
    for (Index j = 0; j < model_.num_cols(); ++j) status_[j] = static_cast<char>(basis_.status[j]);
  }

  cclp::SimplexResult run() {  // :136-153
    cclp::SimplexResult res;
    try {
      res.status = iterate();
    } catch (const cclp::SingularBasisError&) {
      res.status = cclp::SimplexStatus::kNumericalError;
    }
    res.basis = basis_;
    res.pivots = pivots_;
    res.phase1_pivots = phase1_pivots_;
    res.bound_flips = flips_;
    res.refactorizations = refactor_count_;
    res.max_basic_drift = max_drift_;
    res.seconds = elapsed();
    res.iterate = final_iterate();
    return res;
  }

 private:
  Scalar elapsed() const { return std::chrono::duration<double>(Clock::now() - t0_).count(); }

  void set_status(Index j, ColStatus s) {
    basis_.status[j] = s;
    status_[j] = static_cast<char>(s);
  }

  // :162-175; a singular basis swaps its dependent columns for the
  // logicals of the unpivoted rows (sparse rank-revealing repair instead of
  // the dense dependent_positions) and retries once
  void refactorize() {
    std::vector<Index> dep;
    std::vector<int> free_rows;
    if (!factor_.factorize(basis_.basic, &dep, &free_rows)) {
      std::set<Index> basic_set(basis_.basic.begin(), basis_.basic.end());
      size_t fr = 0;
      for (Index pos : dep) {
        while (fr < free_rows.size() && basic_set.count(model_.num_structural() + free_rows[fr])) ++fr;
        if (fr >= free_rows.size()) throw cclp::SingularBasisError("basis repair ran out of logicals", {});
        const Index out = basis_.basic[pos];
        const Index in = model_.num_structural() + free_rows[fr++];
        basis_.basic[pos] = in;
        set_status(out, cclp::default_status(model_, out));
        set_status(in, ColStatus::kBasic);
        x_[out] = basis_.nonbasic_value(model_, out);
      }
      if (!factor_.factorize(basis_.basic, &dep, &free_rows))
        throw cclp::SingularBasisError("unrepairable basis", {});
    }
    ++refactor_count_;
    since_refactor_ = 0;
    if (stats_) stats_->lu_nnz = factor_.nnz();
    recompute_basics();
  }

  void recompute_basics() {  // :202-222
    const Index m = model_.num_rows();
    std::vector<double> r(lp_.row_lower.data(), lp_.row_lower.data() + m);
    for (Index j = 0; j < model_.num_cols(); ++j)
      if (basis_.status[j] != ColStatus::kBasic && x_[j] != 0.0) {
        const double mult = -x_[j];
        cols_.each(j, [&](int i, double v) { r[i] += mult * v; });
      }
    factor_.ftran(r);
    if (basics_valid_) {
      Scalar drift = 0.0;
      for (Index k = 0; k < m; ++k) drift = std::max(drift, std::abs(r[k] - x_[basis_.basic[k]]));
      max_drift_ = std::max(max_drift_, drift);
    }
    for (Index k = 0; k < m; ++k) x_[basis_.basic[k]] = r[k];
    basics_valid_ = true;
  }

  bool infeasibility_gradient(std::vector<double>& g) const {  // :226-247
    const Index m = model_.num_rows();
    g.assign(m, 0.0);
    bool any = false;
    for (Index k = 0; k < m; ++k) {
      const Index j = basis_.basic[k];
      const Scalar below = model_.lower(j) - x_[j];
      const Scalar above = x_[j] - model_.upper(j);
      if (below > ftol_) {
        g[k] = -1.0;
        any = true;
      } else if (above > ftol_) {
        g[k] = 1.0;
        any = true;
      }
    }
    return any;
  }

  struct Pick {
    Index entering = -1;
    int direction = 0;
    Scalar violation = 0.0;
  };

  // :264-296 on the device (the same pick) or on the host
  Pick price(bool phase1, const std::vector<double>& y) {
    Pick pick;
    if (pricer_ != nullptr) {
      long long e = -1;
      int d = 0;
      double v = 0.0;
      pricer_->price(y.data(), status_.data(), skip_any_ ? skip_.data() : nullptr, phase1, dtol_, bland_, &e, &d,
                     &v);
      if (stats_) ++stats_->device_prices;
      if (e >= 0) pick = {static_cast<Index>(e), d, v};
      return pick;
    }
    if (stats_) ++stats_->host_prices;
    for (Index j = 0; j < model_.num_cols(); ++j) {
      const ColStatus st = basis_.status[j];
      if (st == ColStatus::kBasic || st == ColStatus::kFixed) continue;
      if (skip_any_ && skip_[j]) continue;
      const Scalar cost = phase1 ? 0.0 : model_.cost(j);
      double dot = 0.0;
      cols_.each(j, [&](int i, double v) { dot += v * y[i]; });
      const Scalar d = cost - dot;
      Scalar viol = 0.0;
      int dir = 0;
      if (st == ColStatus::kAtLower && d < -dtol_) {
        viol = -d;
        dir = 1;
      } else if (st == ColStatus::kAtUpper && d > dtol_) {
        viol = d;
        dir = -1;
      } else if (st == ColStatus::kFreeAtZero && std::abs(d) > dtol_) {
        viol = std::abs(d);
        dir = d < 0.0 ? 1 : -1;
      } else {
        continue;
      }
      if (bland_) {
        if (pick.entering < 0) pick = {j, dir, viol};
      } else if (viol > pick.violation) {
        pick = {j, dir, viol};
      }
    }
    return pick;
  }

  std::vector<double> basic_costs() const {  // :364-370
    std::vector<double> cb(model_.num_rows());
    for (Index k = 0; k < model_.num_rows(); ++k) cb[k] = model_.cost(basis_.basic[k]);
    return cb;
  }

  cclp::SimplexStatus iterate() {  // :298-362
    refactorize();
    skip_.assign(model_.num_cols(), 0);
    skip_any_ = false;
    std::vector<double> g;
    Vector wv(model_.num_rows());
    while (true) {
      if (opt_.cancel != nullptr && opt_.cancel->load(std::memory_order_relaxed))
        return cclp::SimplexStatus::kCancelled;
      if (elapsed() > opt_.time_limit) return cclp::SimplexStatus::kTimeLimit;
      if (since_refactor_ >= opt_.refactor_interval) refactorize();

      const bool phase1 = infeasibility_gradient(g);
      std::vector<double> y = phase1 ? g : basic_costs();
      factor_.btran(y);
      const Pick pick = price(phase1, y);
      if (pick.entering < 0) return phase1 ? cclp::SimplexStatus::kInfeasible : cclp::SimplexStatus::kOptimal;

      std::vector<double> a(model_.num_rows(), 0.0);
      cols_.each(pick.entering, [&](int i, double v) { a[i] += v; });
      factor_.ftran(a);
      for (Index k = 0; k < model_.num_rows(); ++k) wv[k] = a[k];
      const cclp::RatioOutcome ratio =
          cclp::ratio_test(model_, basis_, x_, pick.entering, pick.direction, wv, ftol_, bland_);
      if (ratio.kind == cclp::RatioOutcome::kUnbounded)
        return phase1 ? cclp::SimplexStatus::kNumericalError : cclp::SimplexStatus::kUnbounded;
      if (pivots_ >= opt_.max_pivots) return cclp::SimplexStatus::kIterationLimit;
      if (ratio.kind == cclp::RatioOutcome::kLeaves && std::abs(a[ratio.leaving_pos]) < kPivotTol) {
        if (factor_.updates() > 0) {
          refactorize();
        } else {
          skip_[pick.entering] = 1;
          skip_any_ = true;
        }
        continue;
      }
      if (skip_any_) {
        std::fill(skip_.begin(), skip_.end(), 0);
        skip_any_ = false;
      }
      apply(pick, a, ratio, phase1);
    }
  }

  void apply(const Pick& pick, const std::vector<double>& w, const cclp::RatioOutcome& ratio, bool phase1) {
    const Scalar t = ratio.step;  // :379-418
    ++pivots_;
    if (phase1) ++phase1_pivots_;
    if (t <= kDegenerateStep) {
      if (++consecutive_degenerate_ > opt_.degenerate_switch) bland_ = true;
    } else {
      consecutive_degenerate_ = 0;
      bland_ = false;
    }
    if (t != 0.0) {
      for (Index k = 0; k < model_.num_rows(); ++k) x_[basis_.basic[k]] -= pick.direction * t * w[k];
      x_[pick.entering] += pick.direction * t;
    }
    if (ratio.kind == cclp::RatioOutcome::kBoundFlip) {
      ++flips_;
      set_status(pick.entering, basis_.status[pick.entering] == ColStatus::kAtUpper ? ColStatus::kAtLower
                                                                                    : ColStatus::kAtUpper);
      x_[pick.entering] = basis_.nonbasic_value(model_, pick.entering);
      return;
    }
    const Index p = ratio.leaving_pos;
    const Index leaving = basis_.basic[p];
    set_status(leaving, ratio.leaving_to);
    x_[leaving] = basis_.nonbasic_value(model_, leaving);
    basis_.basic[p] = pick.entering;
    set_status(pick.entering, ColStatus::kBasic);
    factor_.update(p, w);
    ++since_refactor_;
  }

  cclp::Iterate final_iterate() {  // :420-433
    cclp::Iterate it;
    const Index n = model_.num_structural();
    it.x = x_.head(n);
    std::vector<double> y = basic_costs();
    if (refactor_count_ > 0) {
      factor_.btran(y);
    } else {
      std::fill(y.begin(), y.end(), 0.0);
    }
    it.y = Vector(model_.num_rows());
    for (Index i = 0; i < model_.num_rows(); ++i) it.y[i] = y[i];
    it.z = lp_.c - Vector(lp_.A.transpose() * it.y);
    it.k = pivots_;
    return it;
  }

  EngineModel model_;
  const LinearProgram& lp_;
  Cols cols_;
  cclp::SimplexOptions opt_;
  Basis basis_;
  DevicePricer* pricer_;
  ScalableStats* stats_;
  SparseBasis factor_;
  Vector x_;
  std::vector<char> status_;
  std::vector<unsigned char> skip_;
  bool skip_any_ = false;
  Scalar ftol_ = 1e-9, dtol_ = 1e-9;
  std::int64_t pivots_ = 0, phase1_pivots_ = 0, flips_ = 0;
  int since_refactor_ = 0, refactor_count_ = 0, consecutive_degenerate_ = 0;
  bool bland_ = false, basics_valid_ = false;
  Scalar max_drift_ = 0.0;
  Clock::time_point t0_;
};

cclp::CrossoverStatus from_simplex(cclp::SimplexStatus s) {  // crossover.cpp:224-243
  switch (s) {
    case cclp::SimplexStatus::kOptimal: return cclp::CrossoverStatus::kSuccess;
    case cclp::SimplexStatus::kIterationLimit: return cclp::CrossoverStatus::kIterationLimit;
    case cclp::SimplexStatus::kCancelled: return cclp::CrossoverStatus::kCancelled;
    case cclp::SimplexStatus::kTimeLimit: return cclp::CrossoverStatus::kTimeLimit;
    case cclp::SimplexStatus::kInfeasible: return cclp::CrossoverStatus::kInfeasible;
    case cclp::SimplexStatus::kUnbounded: return cclp::CrossoverStatus::kUnbounded;
    case cclp::SimplexStatus::kNumericalError: return cclp::CrossoverStatus::kNumericalError;
  }
  return cclp::CrossoverStatus::kNumericalError;
}

}  // namespace

// build_basis (crossover.cpp:101-150): statuses of the snapped columns, then
// the candidates in rank order through the incremental sparse LU.
Basis build_basis(const LinearProgram& std_lp, const cclp::Partition& partition, ScalableStats* stats) {
  EngineModel model(std_lp);
  const Index m = model.num_rows();
  Basis basis = cclp::slack_basis(model);
  for (Index j = 0; j < model.num_cols(); ++j) {  // :106-126
    if (basis.status[j] == ColStatus::kBasic) continue;
    switch (partition.label[j]) {
      case cclp::PartitionLabel::kAtLower:
        basis.status[j] = model.lower(j) == model.upper(j)
                              ? ColStatus::kFixed
                              : (cclp::is_finite(model.lower(j)) ? ColStatus::kAtLower
                                                                 : cclp::default_status(model, j));
        break;
      case cclp::PartitionLabel::kAtUpper:
        basis.status[j] = cclp::is_finite(model.upper(j)) ? ColStatus::kAtUpper : cclp::default_status(model, j);
        break;
      case cclp::PartitionLabel::kCandidateBasic:
        basis.status[j] = cclp::default_status(model, j);
        break;
    }
  }
  if (m == 0) return basis;
  const Cols cols = cols_of(std_lp);
  CrashLU lu(static_cast<int>(m));
  Index remaining = m;
  long long offered = 0;
  for (Index j : partition.candidates) {  // :129-146
    if (remaining == 0) break;
    ++offered;
    const int best = lu.offer(cols, j);
    if (best < 0) continue;
    const Index out = basis.basic[best];
    basis.status[out] = cclp::default_status(model, out);
    basis.basic[best] = j;
    basis.status[j] = ColStatus::kBasic;
    --remaining;
  }
  if (stats) {
    stats->crash_candidates = offered;
    stats->crash_accepted = m - remaining;
    stats->lu_nnz = lu.nnz();
  }
  basis.validate(model);
  return basis;
}

// run_crossover (crossover.cpp:247-285) over the scalable pieces.
cclp::CrossoverResult run_crossover(const cclp::CrossoverTask& task, DevicePricer* pricer, ScalableStats* stats) {
  const auto t0 = Clock::now();
  auto since = [](Clock::time_point a) { return std::chrono::duration<double>(Clock::now() - a).count(); };
  ScalableStats local;
  ScalableStats* st = stats ? stats : &local;
  cclp::CrossoverResult res;
  res.launch_threshold = task.launch_threshold;
  const LinearProgram& lp = *task.std_lp;

  auto tc = Clock::now();
  const cclp::Partition part = cclp::guess_partition(lp, task.snapshot, task.launch_threshold);
  const Basis start = build_basis(lp, part, st);
  st->crash_s = since(tc);

  cclp::SimplexOptions opts = task.simplex;
  opts.eps_abs = task.tol.eps_abs;
  tc = Clock::now();
  Simplex engine(lp, start, opts, pricer, st);
  const cclp::SimplexResult cleaned = engine.run();
  st->simplex_s = since(tc);
  res.cleanup_pivots = cleaned.pivots;
  res.basis = cleaned.basis;
  res.status = from_simplex(cleaned.status);
  if (res.status != cclp::CrossoverStatus::kSuccess) {
    res.iterate = cleaned.iterate;
    res.seconds = since(t0);
    return res;
  }
  tc = Clock::now();
  const cclp::VerifyOutcome verdict = cclp::verify_basic_optimal(lp, cleaned.basis, task.tol.eps_abs);
  st->verify_s = since(tc);
  if (!verdict.ok) {
    res.status = cclp::CrossoverStatus::kVerifyFailed;
    res.iterate = cleaned.iterate;
    res.abs_violation = verdict.violation;
    res.seconds = since(t0);
    return res;
  }
  res.iterate = verdict.iterate;
  res.abs_violation = cclp::absolute_violation(lp, res.iterate);
  res.seconds = since(t0);
  return res;
}

}  // namespace cclp_xo
