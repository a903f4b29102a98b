// C-ABI bridge to cclp::run_race (integration/run_race.cpp) for the Python
// tests, the CLI and the time-to-basic benchmark. Built by integration/Makefile twice from
// the same sources: librace_gpu.so (run_pdhg = the B200 drop-in,
// integration/run_pdhg_cuda.cpp) and librace_cpu.so (run_pdhg = the
// reference's own CPU loop). Crossover is the reference's run_crossover in
// both, compiled from /root/reference, so the two differ only in the PDHG.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include <fstream>
#include <memory>

#include "cclp/mps.hpp"
#include "cclp/race.hpp"
#include "crossover_scalable.hpp"
#include "json.hpp"

namespace {
thread_local std::string g_err;

cclp::Vector vec(const double* p, int n) {
  cclp::Vector v(n);
  if (n > 0) std::memcpy(v.data(), p, sizeof(double) * static_cast<size_t>(n));
  return v;
}

// Binary CSC ingest (layout: paper_2510_24429_b200/lp.py, magic "CCLPCSC1"):
// the general-form LP with row activity bounds; the row sense (only used by
// write_mps, mps.cpp:465) follows the bounds.
cclp::LinearProgram read_cscb_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::invalid_argument("cannot open " + path);
  char head[32];
  if (!f.read(head, 32) || std::memcmp(head, "CCLPCSC1", 8) != 0)
    throw std::invalid_argument(path + ": not a CCLPCSC1 file");
  int32_t mn[2];
  int64_t nnz;
  std::memcpy(mn, head + 8, sizeof mn);
  std::memcpy(&nnz, head + 16, sizeof nnz);
  const int m = mn[0], n = mn[1];
  if (m < 0 || n < 0 || nnz < 0) throw std::invalid_argument(path + ": bad header");
  long long off = 32;
  auto read = [&](void* dst, size_t bytes) {
    f.seekg(off);
    if (bytes && !f.read(static_cast<char*>(dst), static_cast<std::streamsize>(bytes)))
      throw std::invalid_argument(path + ": truncated file");
    off = (off + static_cast<long long>(bytes) + 7) / 8 * 8;
  };
  std::vector<int> colptr(static_cast<size_t>(n) + 1), rowind(static_cast<size_t>(nnz));
  std::vector<double> val(static_cast<size_t>(nnz));
  cclp::LinearProgram lp;
  lp.c.resize(n);
  lp.row_lower.resize(m);
  lp.row_upper.resize(m);
  lp.col_lower.resize(n);
  lp.col_upper.resize(n);
  read(colptr.data(), sizeof(int) * colptr.size());
  read(rowind.data(), sizeof(int) * rowind.size());
  read(val.data(), sizeof(double) * val.size());
  read(lp.c.data(), sizeof(double) * n);
  read(lp.row_lower.data(), sizeof(double) * m);
  read(lp.row_upper.data(), sizeof(double) * m);
  read(lp.col_lower.data(), sizeof(double) * n);
  read(lp.col_upper.data(), sizeof(double) * n);
  if (colptr[static_cast<size_t>(n)] != nnz) throw std::invalid_argument(path + ": colptr[n] != nnz");
  lp.A = cclp::SparseMat(Eigen::Map<cclp::SparseMat>(m, n, static_cast<int>(nnz), colptr.data(),
                                                     rowind.data(), val.data()));
  lp.sense.resize(static_cast<size_t>(m));
  for (int i = 0; i < m; ++i) {
    const double l = lp.row_lower[i], u = lp.row_upper[i];
    lp.sense[static_cast<size_t>(i)] =
        l == u ? cclp::RowSense::kEq : (std::isfinite(u) ? cclp::RowSense::kLe : cclp::RowSense::kGe);
  }
  const size_t slash = path.find_last_of('/');
  lp.name = path.substr(slash == std::string::npos ? 0 : slash + 1);
  lp.objective_name = "OBJ";
  lp.validate();
  return lp;
}

bool ends_with(const std::string& s, const char* suf) {
  const size_t k = std::strlen(suf);
  return s.size() >= k && s.compare(s.size() - k, k, suf) == 0;
}
}  // namespace

namespace cclp {
StandardFormMap to_standard_form_direct(const LinearProgram& lp);
}

namespace cclp_race {
extern std::atomic<int> g_crossover, g_device;
extern std::atomic<long long> g_device_prices, g_host_prices;
}  // namespace cclp_race

extern "C" {

const char* cclp_race_last_error() { return g_err.c_str(); }

// The race's crossover: 0 the reference's run_crossover, 1 the scalable one
// with host pricing, 2 the scalable one with pricing on the B200 (device).
// Returns 0, or 1 when kind 2 is asked of a library without the engine.
int cclp_race_set_crossover(int kind, int device) {
#ifdef CCLP_XO_NO_DEVICE
  if (kind == 2) {
    g_err = "cclp_race_set_crossover: this library has no B200 engine (device pricing)";
    return 1;
  }
#endif
  cclp_race::g_crossover.store(kind);
  cclp_race::g_device.store(device);
  return 0;
}
int cclp_race_get_crossover() { return cclp_race::g_crossover.load(); }

// One crossover (crossover.hpp:61-85) on an equality-form LP from a given
// iterate (the snapshot x, y, z in that space), timed: kind as
// cclp_race_set_crossover. `out` receives the result JSON (status, sorted
// basic set, objective, pivots, seconds and the scalable engine's stats).
int cclp_race_crossover(int m, int n, const int* colptr, const int* rowind, const double* val, const double* c,
                        const double* b, const double* cl, const double* cu, const double* x, const double* y,
                        const double* z, double threshold, double eps_abs, int kind, int device, char* out,
                        int cap) {
  try {
    cclp::LinearProgram lp;
    lp.A = cclp::SparseMat(Eigen::Map<cclp::SparseMat>(m, n, colptr[n], colptr, rowind, val));
    lp.c = vec(c, n);
    lp.row_lower = vec(b, m);
    lp.row_upper = vec(b, m);
    lp.col_lower = vec(cl, n);
    lp.col_upper = vec(cu, n);
    lp.sense.assign(static_cast<size_t>(m), cclp::RowSense::kEq);
    cclp::CrossoverTask task;
    task.std_lp = &lp;
    task.snapshot.x = vec(x, n);
    task.snapshot.y = vec(y, m);
    task.snapshot.z = vec(z, n);
    task.launch_threshold = threshold;
    task.tol.eps_abs = eps_abs;
    cclp_xo::ScalableStats st;
    double pricer_s = 0.0;
    const auto t0 = std::chrono::steady_clock::now();
    cclp::CrossoverResult r;
    if (kind == 0) {
      r = cclp::run_crossover(task);
    } else {
      std::unique_ptr<cclp_xo::DevicePricer> pricer;
      if (kind == 2) {
        const auto tp = std::chrono::steady_clock::now();
        pricer = std::make_unique<cclp_xo::DevicePricer>(lp, device);
        pricer_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - tp).count();
      }
      r = cclp_xo::run_crossover(task, pricer.get(), &st);
    }
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<long long> basic(r.basis.basic.begin(), r.basis.basic.end());
    std::sort(basic.begin(), basic.end());
    double obj = 0.0;
    for (int j = 0; j < n && r.iterate.x.size() == n; ++j) obj += lp.c[j] * r.iterate.x[j];
    nlohmann::json j{{"status", cclp::to_string(r.status)}, {"basic", basic}, {"objective", obj},
                     {"pivots", r.cleanup_pivots}, {"seconds", r.seconds}, {"wall_s", wall},
                     {"pricer_setup_s", pricer_s}, {"violation", r.abs_violation},
                     {"crash_candidates", st.crash_candidates}, {"crash_accepted", st.crash_accepted},
                     {"lu_nnz", st.lu_nnz}, {"device_prices", st.device_prices},
                     {"host_prices", st.host_prices}, {"crash_s", st.crash_s}, {"simplex_s", st.simplex_s},
                     {"verify_s", st.verify_s}};
    const std::string s2 = j.dump();
    if (static_cast<int>(s2.size()) + 1 > cap) {
      g_err = "cclp_race_crossover: output buffer too small";
      return 2;
    }
    std::memcpy(out, s2.c_str(), s2.size() + 1);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
// Pricing calls made by scalable crossovers since load: [0] device, [1] host.
void cclp_race_pricing_counts(long long* out) {
  out[0] = cclp_race::g_device_prices.load();
  out[1] = cclp_race::g_host_prices.load();
}

// mode 0 = baseline, 1 = concurrent. Writes the RaceOutcome JSON plus the
// sorted basic column set and the event log into `out` (NUL-terminated).
int cclp_race_run(int m, int n, const int* colptr, const int* rowind, const double* val, const double* c,
                  const double* rl, const double* ru, const double* cl, const double* cu, int mode,
                  double eps_rel, double eps_cross, double eps_abs, double time_limit, int pool,
                  long long max_iterations, char* out, int cap) {
  try {
    cclp::LinearProgram lp;
    lp.A = cclp::SparseMat(Eigen::Map<cclp::SparseMat>(m, n, colptr[n], colptr, rowind, val));
    lp.c = vec(c, n);
    lp.row_lower = vec(rl, m);
    lp.row_upper = vec(ru, m);
    lp.col_lower = vec(cl, n);
    lp.col_upper = vec(cu, n);
    lp.sense.assign(static_cast<size_t>(m), cclp::RowSense::kEq);
    for (int i = 0; i < m; ++i)
      if (rl[i] != ru[i]) lp.sense[static_cast<size_t>(i)] = cclp::RowSense::kLe;
    cclp::RaceConfig cfg;
    cfg.mode = mode ? cclp::RaceMode::kConcurrent : cclp::RaceMode::kBaseline;
    cfg.tol.eps_rel = eps_rel;
    cfg.tol.eps_cross = eps_cross;
    cfg.tol.eps_abs = eps_abs;
    cfg.time_limit = time_limit;
    cfg.worker_pool = pool;
    cfg.pdhg.max_iterations = max_iterations;
    std::ostringstream events;
    cfg.event_log = &events;
    cclp::RaceOutcome o = cclp::run_race(lp, cfg);
    nlohmann::json j = nlohmann::json::parse(o.to_json());
    std::vector<long long> basic(o.final_result.basis.basic.begin(), o.final_result.basis.basic.end());
    std::sort(basic.begin(), basic.end());
    j["basic"] = basic;
    j["winning_threshold"] = o.winning_threshold;
    j["thresholds"] = o.thresholds;
    j["events"] = events.str();
    j["x"] = std::vector<double>(o.solution.x.data(), o.solution.x.data() + o.solution.x.size());
    const std::string s = j.dump();
    if (static_cast<int>(s.size()) + 1 > cap) {
      g_err = "cclp_race_run: output buffer too small (" + std::to_string(s.size() + 1) + ")";
      return 2;
    }
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// `solve <model.mps>` (SPEC bench_cli): read_mps_file -> run_race, then the
// basis (write_basis, basis.hpp:92) and the solution file (objective header,
// then "column value status" per line) when paths are given. Returns the SPEC
// exit code: 0 solved, 2 time limit, 3 numerical failure / unsolved, 4 input
// error; `out` receives the outcome JSON.
int cclp_race_solve_file(const char* path, int mode, double eps_rel, double eps_cross, double eps_abs,
                         double decrement, int pool, double time_limit, unsigned long long seed,
                         const char* basis_out, const char* solution_out, char* out, int cap) {
  cclp::LinearProgram lp;
  try {
    lp = ends_with(path, ".cscb") ? read_cscb_file(path) : cclp::read_mps_file(path);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
  try {
    cclp::RaceConfig cfg;
    cfg.mode = mode ? cclp::RaceMode::kConcurrent : cclp::RaceMode::kBaseline;
    cfg.tol.eps_rel = eps_rel;
    cfg.tol.eps_cross = eps_cross;
    cfg.tol.eps_abs = eps_abs;
    cfg.tol.decrement = decrement;
    cfg.worker_pool = pool;
    cfg.time_limit = time_limit;
    cfg.pdhg.seed = seed;
    std::ostringstream events;
    cfg.event_log = &events;
    cclp::RaceOutcome o = cclp::run_race(lp, cfg);
    nlohmann::json j = nlohmann::json::parse(o.to_json());
    j["model"] = lp.name;
    j["rows"] = lp.num_rows();
    j["cols"] = lp.num_cols();
    j["winning_threshold"] = o.winning_threshold;
    std::int64_t pivots = o.final_result.cleanup_pivots;
    j["pivots"] = pivots;
    j["violation"] = o.final_result.abs_violation;
    j["events"] = events.str();
    if (o.status == cclp::RaceStatus::kSolved) {
      const cclp::StandardFormMap sf = cclp::to_standard_form_direct(lp);
      if (basis_out && *basis_out) {
        std::ofstream f(basis_out);
        cclp::write_basis(cclp::EngineModel(sf.std_lp), o.final_result.basis, f);
      }
      if (solution_out && *solution_out) {
        std::ofstream f(solution_out);
        char line[256];
        std::snprintf(line, sizeof line, "* objective %.17g\n", o.objective);
        f << line;
        std::vector<bool> basic(static_cast<size_t>(sf.std_lp.num_cols()), false);
        for (auto jb : o.final_result.basis.basic)
          if (jb < sf.std_lp.num_cols()) basic[static_cast<size_t>(jb)] = true;
        for (cclp::Index jc = 0; jc < lp.num_cols(); ++jc) {
          const std::string name = jc < static_cast<cclp::Index>(lp.col_names.size())
                                       ? lp.col_names[static_cast<size_t>(jc)]
                                       : "C" + std::to_string(jc);
          const char* st = basic[static_cast<size_t>(jc)] ? "basic" : "nonbasic";
          std::snprintf(line, sizeof line, "%s %.17g %s\n", name.c_str(), o.solution.x[jc], st);
          f << line;
        }
      }
    }
    const std::string str = j.dump();
    if (static_cast<int>(str.size()) + 1 > cap) {
      g_err = "cclp_race_solve_file: output buffer too small";
      return 4;
    }
    std::memcpy(out, str.c_str(), str.size() + 1);
    switch (o.status) {
      case cclp::RaceStatus::kSolved: return 0;
      case cclp::RaceStatus::kTimeLimit: return 2;
      default: return 3;
    }
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

// write_mps (mps.hpp:50) of an LP given as arrays (rows named R<i>, columns
// C<j>, equality rows where lower == upper): test and bench fixtures.
int cclp_race_write_mps(int m, int n, const int* colptr, const int* rowind, const double* val,
                        const double* c, const double* rl, const double* ru, const double* cl,
                        const double* cu, const char* name, const char* path) {
  try {
    cclp::LinearProgram lp;
    lp.name = name ? name : "LP";
    lp.objective_name = "OBJ";
    lp.A = cclp::SparseMat(Eigen::Map<cclp::SparseMat>(m, n, colptr[n], colptr, rowind, val));
    lp.c = vec(c, n);
    lp.row_lower = vec(rl, m);
    lp.row_upper = vec(ru, m);
    lp.col_lower = vec(cl, n);
    lp.col_upper = vec(cu, n);
    lp.sense.assign(static_cast<size_t>(m), cclp::RowSense::kEq);
    for (int i = 0; i < m; ++i) {
      if (rl[i] == ru[i]) continue;
      lp.sense[static_cast<size_t>(i)] = std::isfinite(ru[i]) ? cclp::RowSense::kLe : cclp::RowSense::kGe;
    }
    for (int i = 0; i < m; ++i) lp.row_names.push_back("R" + std::to_string(i));
    for (int j = 0; j < n; ++j) lp.col_names.push_back("C" + std::to_string(j));
    std::ofstream f(path);
    cclp::write_mps(lp, f);
    return f.good() ? 0 : 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Host-only helpers with the reference's semantics (race.hpp:86-100).
int cclp_race_schedule(double eps_rel, double eps_cross, double decrement, double* out, int cap) {
  try {
    cclp::Tolerances t;
    t.eps_rel = eps_rel;
    t.eps_cross = eps_cross;
    t.decrement = decrement;
    const auto v = cclp::schedule_thresholds(t);
    for (int i = 0; i < cap && i < static_cast<int>(v.size()); ++i) out[i] = v[static_cast<size_t>(i)];
    return static_cast<int>(v.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void cclp_race_reserve(int pool, int cores, int* pdhg, int* crossover) {
  cclp::RaceConfig cfg;
  cfg.worker_pool = pool;
  const auto p = cclp::reserve_threads(cfg, cores);
  *pdhg = p.first;
  *crossover = p.second;
}

// run_race_simulated on a scripted trace: workers given as parallel arrays.
int cclp_race_simulate(const double* trace, int ntrace, double sec_per_iter, const double* thr,
                       const double* dur, const int* verifies, int nworkers, double main_dur, int main_ok,
                       int mode, double eps_rel, double eps_cross, int pool, double time_limit, char* out,
                       int cap) {
  try {
    cclp::RaceScript script;
    script.residual_trace.assign(trace, trace + ntrace);
    script.seconds_per_iteration = sec_per_iter;
    for (int i = 0; i < nworkers; ++i) script.workers[thr[i]] = cclp::SimWorker{dur[i], verifies[i] != 0};
    script.main_worker = cclp::SimWorker{main_dur, main_ok != 0};
    cclp::RaceConfig cfg;
    cfg.mode = mode ? cclp::RaceMode::kConcurrent : cclp::RaceMode::kBaseline;
    cfg.tol.eps_rel = eps_rel;
    cfg.tol.eps_cross = eps_cross;
    cfg.worker_pool = pool;
    cfg.time_limit = time_limit;
    std::ostringstream events;
    cfg.event_log = &events;
    cclp::RaceOutcome o = cclp::run_race_simulated(script, cfg);
    nlohmann::json j = nlohmann::json::parse(o.to_json());
    j["winning_threshold"] = o.winning_threshold;
    j["events"] = events.str();
    const std::string s = j.dump();
    if (static_cast<int>(s.size()) + 1 > cap) return 2;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}


// Test hook: the race's O(nnz) standard form against the reference's
// to_standard_form on the same LP (row senses from the bounds, optional max
// objective). 0 = identical in every field, 1 = differs (reason in
// cclp_race_last_error), 2 = error. seconds (optional) receives the two
// wall times {reference, direct}.
int cclp_race_standard_form_check(int m, int n, const int* colptr, const int* rowind, const double* val,
                                  const double* c, const double* rl, const double* ru, const double* cl,
                                  const double* cu, int maximize, int named, double* seconds) {
  try {
    cclp::LinearProgram lp;
    lp.A = cclp::SparseMat(Eigen::Map<cclp::SparseMat>(m, n, colptr[n], colptr, rowind, val));
    lp.c = vec(c, n);
    lp.row_lower = vec(rl, m);
    lp.row_upper = vec(ru, m);
    lp.col_lower = vec(cl, n);
    lp.col_upper = vec(cu, n);
    lp.obj_sense = maximize ? cclp::ObjSense::kMax : cclp::ObjSense::kMin;
    lp.obj_offset = 1.25;
    lp.sense.resize(static_cast<size_t>(m));
    for (int i = 0; i < m; ++i)
      lp.sense[static_cast<size_t>(i)] =
          rl[i] == ru[i] ? cclp::RowSense::kEq : (std::isfinite(ru[i]) ? cclp::RowSense::kLe : cclp::RowSense::kGe);
    if (named) {
      for (int i = 0; i < m; ++i) lp.row_names.push_back("row" + std::to_string(i));
      for (int j = 0; j < n; ++j) lp.col_names.push_back("col" + std::to_string(j));
    }
    const auto t0 = std::chrono::steady_clock::now();
    const cclp::StandardFormMap a = cclp::to_standard_form(lp);
    const auto t1 = std::chrono::steady_clock::now();
    const cclp::StandardFormMap b = cclp::to_standard_form_direct(lp);
    const auto t2 = std::chrono::steady_clock::now();
    if (seconds) {
      seconds[0] = std::chrono::duration<double>(t1 - t0).count();
      seconds[1] = std::chrono::duration<double>(t2 - t1).count();
    }
    auto vec_eq = [](const cclp::Vector& x, const cclp::Vector& y) {
      if (x.size() != y.size()) return false;
      for (cclp::Index i = 0; i < x.size(); ++i)
        if (std::memcmp(x.data() + i, y.data() + i, sizeof(double)) != 0) return false;
      return true;
    };
    const auto& A = a.std_lp.A;
    const auto& B = b.std_lp.A;
    std::string why;
    if (A.rows() != B.rows() || A.cols() != B.cols() || A.nonZeros() != B.nonZeros()) why = "A shape";
    else if (!std::equal(A.outerIndexPtr(), A.outerIndexPtr() + A.cols() + 1, B.outerIndexPtr())) why = "A colptr";
    else if (!std::equal(A.innerIndexPtr(), A.innerIndexPtr() + A.nonZeros(), B.innerIndexPtr())) why = "A rowind";
    else if (std::memcmp(A.valuePtr(), B.valuePtr(), sizeof(double) * static_cast<size_t>(A.nonZeros())) != 0)
      why = "A values";
    else if (!vec_eq(a.std_lp.c, b.std_lp.c)) why = "c";
    else if (!vec_eq(a.std_lp.row_lower, b.std_lp.row_lower) || !vec_eq(a.std_lp.row_upper, b.std_lp.row_upper))
      why = "row bounds";
    else if (!vec_eq(a.std_lp.col_lower, b.std_lp.col_lower) || !vec_eq(a.std_lp.col_upper, b.std_lp.col_upper))
      why = "column bounds";
    else if (a.std_lp.col_names != b.std_lp.col_names || a.std_lp.row_names != b.std_lp.row_names) why = "names";
    else if (a.std_lp.sense != b.std_lp.sense || a.std_lp.obj_sense != b.std_lp.obj_sense ||
             a.std_lp.obj_offset != b.std_lp.obj_offset || a.std_lp.name != b.std_lp.name)
      why = "senses / offset";
    else if (a.slack_col_of_row != b.slack_col_of_row || a.negated != b.negated || a.orig_cols != b.orig_cols ||
             a.orig_rows != b.orig_rows)
      why = "map";
    g_err = why;
    return why.empty() ? 0 : 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // extern "C"
