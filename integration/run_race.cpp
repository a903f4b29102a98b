// cclp::run_race and friends (reference: proj/include/cclp/race.hpp:95-129,
// spec SPEC.md "[MODULE] race"; declared but not implemented upstream):
// Algorithm 1 of the paper over the B200 PDHG. One coordinator thread runs
// run_pdhg with the threshold ladder; every ladder snapshot (delivered by the
// engine's sink, copied to pinned memory on a side stream) launches a CPU
// crossover worker (the reference's run_crossover) if the pool has room; the
// first worker whose basis re-verifies wins, and every other worker, the main
// crossover and the PDHG loop are cancelled. Baseline mode runs PDHG to
// eps_rel and then one crossover on the main thread.
//
// run_pdhg here is whichever definition is linked: the drop-in
// (integration/run_pdhg_cuda.cpp, the GPU engine) or the reference's CPU loop
// - the orchestration is identical, which is how the time-to-basic benchmark
// compares the two.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <limits>
#include <memory>
#include <mutex>
#include <ostream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "cclp/race.hpp"
#include "crossover_scalable.hpp"
#include "json.hpp"

// Which crossover the race's workers and main thread run: the reference's
// run_crossover (dense etas; m up to ~1e4) or the scalable one
// (crossover_scalable.hpp: sparse LU crash and factors, pricing on the B200
// when the library carries the engine). Set through cclp_race_set_crossover.
namespace cclp_race {
#ifdef CCLP_RACE_DEFAULT_SCALABLE
std::atomic<int> g_crossover{2};  // 2: scalable + device pricing
#else
std::atomic<int> g_crossover{0};  // 0: reference
#endif
std::atomic<int> g_device{0};
std::atomic<long long> g_device_prices{0}, g_host_prices{0};
}  // namespace cclp_race

namespace cclp {

// integration/standard_form_direct.cpp: the same map in O(nnz).
StandardFormMap to_standard_form_direct(const LinearProgram& lp);

const char* to_string(RaceStatus status) {
  switch (status) {
    case RaceStatus::kSolved: return "solved";
    case RaceStatus::kTimeLimit: return "time-limit";
    case RaceStatus::kPdhgLimit: return "pdhg-limit";
    case RaceStatus::kNumericalError: return "numerical-error";
    case RaceStatus::kFailed: return "failed";
  }
  return "unknown";
}

void RaceConfig::validate() const {
  tol.validate();
  if (mode == RaceMode::kConcurrent && worker_pool < 1)
    throw std::invalid_argument("race: worker pool must be >= 1 in concurrent mode");
  if (!(time_limit > 0.0)) throw std::invalid_argument("race: time limit must be positive");
}

std::string RaceEvent::to_json() const {
  nlohmann::json j{{"event", event}, {"threshold", label}, {"t_ms", t_ms}};
  if (!status.empty()) j["status"] = status;
  return j.dump();
}

std::string RaceOutcome::to_json() const {
  nlohmann::json workers_j = nlohmann::json::array();
  for (const auto& w : workers)
    workers_j.push_back({{"threshold", threshold_label(w.threshold)},
                         {"launch_s", w.launch_s},
                         {"finish_s", w.finish_s},
                         {"status", to_string(w.status)},
                         {"pivots", w.pivots}});
  nlohmann::json j{{"status", to_string(status)},
                   {"winner", winner_label},
                   {"main_won", main_won},
                   {"objective", objective},
                   {"pdhg_stop", to_string(pdhg_stop)},
                   {"pdhg_iterations", pdhg_iterations},
                   {"wall_s", wall_s},
                   {"workers", workers_j}};
  return j.dump();
}

// eps_cross, eps_cross*decrement, ... while strictly above eps_rel; the
// product runs in extended precision and each value is snapped through a
// 15-digit decimal round trip, so 1e-2 x 0.1 gives exactly 1e-3.
std::vector<Scalar> schedule_thresholds(const Tolerances& tol) {
  tol.validate();
  std::vector<Scalar> out;
  long double t = tol.eps_cross;
  for (int guard = 0; guard < 4096; ++guard) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.15Lg", t);
    const Scalar v = std::strtod(buf, nullptr);
    if (!(v > tol.eps_rel)) break;
    out.push_back(v);
    t *= static_cast<long double>(tol.decrement);
  }
  return out;
}

std::pair<int, int> reserve_threads(const RaceConfig& config, int available_cores) {
  const int avail = std::max(2, available_cores);
  const int pool = std::max(1, std::min(config.worker_pool, avail - 1));
  const int pdhg = config.pdhg_threads > 0 ? config.pdhg_threads : std::max(1, avail - pool);
  return {pdhg, pool};
}

std::string threshold_label(Scalar threshold) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%.0e", threshold);
  return buf;
}

namespace {

using Clock = std::chrono::steady_clock;

// State shared by the coordinator and the workers of one race.
struct RaceState {
  const LinearProgram* std_lp = nullptr;
  const RaceConfig* config = nullptr;
  Clock::time_point t0;
  std::mutex mu;
  bool have_winner = false;
  std::atomic<bool> pdhg_cancel{false};
  std::atomic<bool> main_cancel{false};
  std::atomic<int> running{0};
  RaceOutcome* out = nullptr;

  struct Worker {
    Scalar threshold = 0.0;
    std::string label;
    std::atomic<bool> cancel{false};
    std::thread th;
    WorkerRecord rec;
    bool finished = false;
  };
  std::deque<Worker> workers;  // stable addresses

  double now_s() const { return std::chrono::duration<double>(Clock::now() - t0).count(); }

  void event(const std::string& ev, const std::string& label, const std::string& status = "") {
    RaceEvent e{ev, label, 1e3 * now_s(), status};
    out->events.push_back(e);
    if (config->event_log) *config->event_log << e.to_json() << "\n";
  }

  // Re-verification by the race itself, then an atomic commit: the first
  // verified basis wins; everything else is cancelled.
  bool try_commit(const std::string& label, Scalar threshold, CrossoverResult r, bool main) {
    VerifyOutcome v = verify_basic_optimal(*std_lp, r.basis, config->tol.eps_abs);
    std::lock_guard<std::mutex> g(mu);
    if (!v.ok || have_winner) return false;
    have_winner = true;
    out->main_won = main;
    out->winning_threshold = threshold;
    out->winner_label = label;
    r.iterate = v.iterate;
    out->final_result = std::move(r);
    pdhg_cancel.store(true, std::memory_order_relaxed);
    main_cancel.store(true, std::memory_order_relaxed);
    event("win", label, "success");
    for (auto& w : workers)
      if (!w.finished && w.label != label) {
        w.cancel.store(true, std::memory_order_relaxed);
        event("cancel", w.label);
      }
    return true;
  }

  std::unique_ptr<cclp_xo::DevicePricer> pricer;  // crossover kind 2 only
  CrossoverResult crossover(const CrossoverTask& task) {
    const int kind = cclp_race::g_crossover.load();
    if (kind == 0) return run_crossover(task);
    cclp_xo::ScalableStats st;
    CrossoverResult r = cclp_xo::run_crossover(task, kind == 2 ? pricer.get() : nullptr, &st);
    cclp_race::g_device_prices += st.device_prices;
    cclp_race::g_host_prices += st.host_prices;
    return r;
  }

  CrossoverTask task_for(const Iterate& it, Scalar maxresid, const std::atomic<bool>* cancel) const {
    CrossoverTask task;
    task.std_lp = std_lp;
    task.snapshot = it;
    task.launch_threshold = maxresid;
    task.tol = config->tol;
    task.simplex = config->simplex;
    task.simplex.cancel = cancel;
    task.simplex.time_limit = std::max(0.0, std::min(config->simplex.time_limit, config->time_limit - now_s()));
    return task;
  }

  // The snapshot sink (runs on the PDHG thread; must not block): launch a
  // worker if the pool has room, else drop the snapshot (SPEC: later
  // snapshots are better starting points than queued stale ones).
  void launch(const PdhgSnapshot& snap, int pool) {
    std::lock_guard<std::mutex> g(mu);
    if (have_winner || running.load() >= pool) return;
    workers.emplace_back();
    Worker& w = workers.back();
    w.threshold = snap.threshold;
    w.label = threshold_label(snap.threshold);
    w.rec.threshold = snap.threshold;
    w.rec.launch_s = now_s();
    running.fetch_add(1);
    event("launch", w.label);
    CrossoverTask task = task_for(snap.iterate, snap.maxresid, &w.cancel);
    w.th = std::thread([this, &w, task = std::move(task)]() {
      CrossoverResult r = crossover(task);
      {
        std::lock_guard<std::mutex> g2(mu);
        w.rec.finish_s = now_s();
        w.rec.status = r.status;
        w.rec.pivots = r.cleanup_pivots;
        w.finished = true;
        event("finish", w.label, to_string(r.status));
      }
      if (r.status == CrossoverStatus::kSuccess) try_commit(w.label, w.threshold, std::move(r), false);
      running.fetch_sub(1);
    });
  }
};

}  // namespace

RaceOutcome run_race(const LinearProgram& lp, const RaceConfig& config) {
  config.validate();
  RaceOutcome out;
  RaceState S;
  S.config = &config;
  S.out = &out;
  S.t0 = Clock::now();
  const StandardFormMap sf = to_standard_form_direct(lp);
  S.std_lp = &sf.std_lp;
  if (cclp_race::g_crossover.load() == 2)  // the device pricing context (LP upload, CSR)
    S.pricer = std::make_unique<cclp_xo::DevicePricer>(sf.std_lp, cclp_race::g_device.load());
  const bool concurrent = config.mode == RaceMode::kConcurrent;
  out.thresholds = concurrent ? schedule_thresholds(config.tol) : std::vector<Scalar>{};
  const int pool = reserve_threads(config, static_cast<int>(std::thread::hardware_concurrency())).second;

  PdhgConfig pcfg = config.pdhg;
  pcfg.time_limit = std::min(pcfg.time_limit, config.time_limit);
  S.event("launch", "pdhg");
  SnapshotSink sink = nullptr;
  if (concurrent) sink = [&S, pool](const PdhgSnapshot& s) { S.launch(s, pool); };
  PdhgResult pr = run_pdhg(sf.std_lp, pcfg, config.tol, out.thresholds, sink, &S.pdhg_cancel);
  out.pdhg_stop = pr.stop;
  out.pdhg_iterations = pr.iterations;
  out.pdhg_report = pr.report;
  {
    std::lock_guard<std::mutex> g(S.mu);
    if (S.have_winner && pr.stop == PdhgStopReason::kCancelled) out.pdhg_stop = PdhgStopReason::kWonByCrossover;
    S.event("finish", "pdhg", to_string(out.pdhg_stop));
  }

  // Main-thread crossover from the converged iterate (identical to baseline).
  bool main_ran = false;
  if (pr.stop == PdhgStopReason::kConverged) {
    bool skip;
    {
      std::lock_guard<std::mutex> g(S.mu);
      skip = S.have_winner;
      if (!skip) S.event("launch", "main");
    }
    if (!skip) {
      main_ran = true;
      CrossoverResult r = S.crossover(S.task_for(pr.iterate, pr.report.maxresid_rel, &S.main_cancel));
      {
        std::lock_guard<std::mutex> g(S.mu);
        S.event("finish", "main", to_string(r.status));
      }
      if (r.status == CrossoverStatus::kSuccess) S.try_commit("main", config.tol.eps_rel, std::move(r), true);
    }
  }
  for (auto& w : S.workers)
    if (w.th.joinable()) w.th.join();
  for (auto& w : S.workers) out.workers.push_back(w.rec);

  const double wall = S.now_s();
  if (S.have_winner) {
    out.status = RaceStatus::kSolved;
    const Iterate& it = out.final_result.iterate;
    out.solution.x = sf.drop_x(it.x);
    out.solution.y = sf.drop_y(it.y);
    out.solution.z = sf.drop_z(it.z);
    out.objective = sf.unmap_objective(sf.std_lp.c.dot(it.x));
  } else if (pr.stop == PdhgStopReason::kNumericalError) {
    out.status = RaceStatus::kNumericalError;
  } else if (pr.stop == PdhgStopReason::kTimeLimit || wall >= config.time_limit) {
    out.status = RaceStatus::kTimeLimit;
  } else if (pr.stop == PdhgStopReason::kIterationLimit && !main_ran) {
    out.status = RaceStatus::kPdhgLimit;
  } else {
    out.status = RaceStatus::kFailed;
  }
  out.wall_s = wall;
  return out;
}

// Deterministic simulation of the same rules on a scripted trace: PDHG check
// k happens at k * seconds_per_iteration with maxresid residual_trace[k];
// a check at or below the next ladder threshold emits one snapshot (as
// run_pdhg does, pdhg.cpp:346-358) that launches a scripted worker if fewer
// than `pool` are running; convergence launches the main crossover; the first
// verified finish wins and stops PDHG.
RaceOutcome run_race_simulated(const RaceScript& script, const RaceConfig& config) {
  config.validate();
  RaceOutcome out;
  const bool concurrent = config.mode == RaceMode::kConcurrent;
  out.thresholds = concurrent ? schedule_thresholds(config.tol) : std::vector<Scalar>{};
  const int pool = reserve_threads(config, static_cast<int>(std::thread::hardware_concurrency())).second;
  struct Run {
    std::string label;
    Scalar threshold;
    double launch, finish;
    bool verifies, main;
  };
  std::vector<Run> runs;
  auto log = [&](const std::string& ev, const std::string& label, double t, const std::string& st = "") {
    out.events.push_back(RaceEvent{ev, label, 1e3 * t, st});
    if (config.event_log) *config.event_log << out.events.back().to_json() << "\n";
  };
  // earliest verified finish among the runs launched so far
  auto best_finish = [&]() {
    double b = std::numeric_limits<double>::infinity();
    for (const auto& r : runs)
      if (r.verifies) b = std::min(b, r.finish);
    return b;
  };
  size_t next = 0;
  double pdhg_end = 0.0;
  out.pdhg_stop = PdhgStopReason::kIterationLimit;
  for (size_t k = 0; k < script.residual_trace.size(); ++k) {
    const double t = static_cast<double>(k) * script.seconds_per_iteration;
    if (t >= config.time_limit) {
      out.pdhg_stop = PdhgStopReason::kTimeLimit;
      pdhg_end = config.time_limit;
      break;
    }
    if (t >= best_finish()) {  // a worker already won: PDHG was cancelled
      out.pdhg_stop = PdhgStopReason::kWonByCrossover;
      pdhg_end = best_finish();
      break;
    }
    out.pdhg_iterations = static_cast<std::int64_t>(k);
    const Scalar r = script.residual_trace[k];
    pdhg_end = t;
    if (r <= config.tol.eps_rel) {
      out.pdhg_stop = PdhgStopReason::kConverged;
      runs.push_back({"main", config.tol.eps_rel, t, t + script.main_worker.duration_s,
                      script.main_worker.verifies, true});
      log("launch", "main", t);
      break;
    }
    if (concurrent && next < out.thresholds.size() && r <= out.thresholds[next]) {
      const Scalar thr = out.thresholds[next++];
      int running = 0;
      for (const auto& q : runs)
        if (q.launch <= t && t < q.finish) ++running;
      auto it = script.workers.find(thr);
      if (running < pool && it != script.workers.end()) {
        runs.push_back({threshold_label(thr), thr, t, t + it->second.duration_s, it->second.verifies, false});
        log("launch", threshold_label(thr), t);
      }
    }
  }
  // the winner: first verified finish within the time limit; ties -> launch order
  int win = -1;
  for (size_t i = 0; i < runs.size(); ++i)
    if (runs[i].verifies && runs[i].finish <= config.time_limit &&
        (win < 0 || runs[i].finish < runs[win].finish))
      win = static_cast<int>(i);
  const double t_end = win >= 0 ? runs[win].finish : std::min(config.time_limit, [&] {
    double e = pdhg_end;
    for (const auto& r : runs) e = std::max(e, r.finish);
    return e;
  }());
  for (size_t i = 0; i < runs.size(); ++i) {
    const Run& r = runs[i];
    WorkerRecord rec;
    rec.threshold = r.threshold;
    rec.launch_s = r.launch;
    if (static_cast<int>(i) == win) {
      rec.finish_s = r.finish;
      rec.status = CrossoverStatus::kSuccess;
      log("finish", r.label, r.finish, "success");
      log("win", r.label, r.finish, "success");
    } else if (r.finish <= t_end) {
      rec.finish_s = r.finish;
      rec.status = r.verifies ? CrossoverStatus::kSuccess : CrossoverStatus::kVerifyFailed;
      log("finish", r.label, r.finish, to_string(rec.status));
    } else {
      rec.finish_s = t_end;
      rec.status = CrossoverStatus::kCancelled;
      log("cancel", r.label, t_end);
    }
    if (!r.main) out.workers.push_back(rec);
  }
  std::stable_sort(out.events.begin(), out.events.end(),
                   [](const RaceEvent& a, const RaceEvent& b) { return a.t_ms < b.t_ms; });
  if (win >= 0) {
    out.status = RaceStatus::kSolved;
    out.main_won = runs[win].main;
    out.winner_label = runs[win].label;
    out.winning_threshold = runs[win].threshold;
    if (!out.main_won && out.pdhg_stop != PdhgStopReason::kConverged)
      out.pdhg_stop = PdhgStopReason::kWonByCrossover;
  } else if (out.pdhg_stop == PdhgStopReason::kTimeLimit || t_end >= config.time_limit) {
    out.status = RaceStatus::kTimeLimit;
  } else if (out.pdhg_stop == PdhgStopReason::kIterationLimit) {
    out.status = RaceStatus::kPdhgLimit;
  } else {
    out.status = RaceStatus::kFailed;
  }
  out.wall_s = t_end;
  return out;
}

}  // namespace cclp
