// Drop-in replacement for cclp::run_pdhg (reference: proj/include/cclp/pdhg.hpp:138-142,
// proj/src/pdhg.cpp:230-378) backed by the B200 engine's C ABI (include/cclp_cu.h).
//
// A maintainer adds this file to the reference's library in place of the
// run_pdhg definition in pdhg.cpp (the step-level API — estimate_matrix_norm,
// make_initial_state, pdhg_step, restart_if_improved — stays the reference's
// host code) and links paper_2510_24429_b200/libcclp_cuda.so. The signature,
// argument meaning, exceptions and stop reasons are the reference's:
//   * std::invalid_argument for a non-equality LP, invalid tolerances or
//     non-decreasing thresholds (pdhg.cpp:235-244);
//   * a non-finite iterate is stop reason kNumericalError with
//     error_iteration, not an exception (pdhg.cpp:369-376);
//   * the sink runs on the calling thread (pdhg.cpp:346-358) while the device
//     keeps iterating; an exception it throws stops the loop at the next
//     iteration (cclp_cu_request_cancel) and propagates unchanged out of
//     run_pdhg, as the reference's synchronous call would;
//   * cancel is polled with a relaxed load every iteration (pdhg.cpp:301).
// integration/Makefile links it into librace_gpu.so; oracle/Makefile's `dropin`
// target builds the reference's own test_pdhg.cpp
// against this file (tests/test_dropin.py runs it on the GPU).
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "cclp/pdhg.hpp"
#include "cclp_cu.h"

namespace cclp {

namespace {

struct SinkBridge {
  const SnapshotSink* sink;
  Index m, n;
  cclp_cu_ctx* ctx = nullptr;
  std::exception_ptr error;  // the sink's exception, rethrown after the solve
};

void sink_call(SinkBridge* b, const cclp_cu_snapshot* s);

void sink_trampoline(const cclp_cu_snapshot* s, void* user) {
  auto* b = static_cast<SinkBridge*>(user);
  if (b->sink == nullptr || !*b->sink || b->error) return;
  try {
    sink_call(b, s);
  } catch (...) {  // never unwind through the C ABI
    b->error = std::current_exception();
    cclp_cu_request_cancel(b->ctx);
  }
}

void sink_call(SinkBridge* b, const cclp_cu_snapshot* s) {
  PdhgSnapshot snap;
  snap.iterate.x = Vector(b->n);
  snap.iterate.y = Vector(b->m);
  snap.iterate.z = Vector(b->n);
  if (b->n > 0) {
    std::memcpy(snap.iterate.x.data(), s->x, sizeof(double) * static_cast<size_t>(b->n));
    std::memcpy(snap.iterate.z.data(), s->z, sizeof(double) * static_cast<size_t>(b->n));
  }
  if (b->m > 0) std::memcpy(snap.iterate.y.data(), s->y, sizeof(double) * static_cast<size_t>(b->m));
  snap.iterate.k = s->iteration;
  snap.threshold = s->threshold;
  snap.maxresid = s->maxresid;
  snap.from_average = s->from_average != 0;
  snap.iteration = s->iteration;
  (*b->sink)(snap);
}

void log_trampoline(const char* line, void* user) {
  auto* os = static_cast<std::ostream*>(user);
  (*os) << line << std::flush;
}

}  // namespace

PdhgResult run_pdhg(const LinearProgram& std_lp, const PdhgConfig& config, const Tolerances& tol,
                    const std::vector<Scalar>& thresholds, const SnapshotSink& sink,
                    const std::atomic<bool>* cancel) {
  if (!std_lp.all_rows_equality()) {
    throw std::invalid_argument("run_pdhg: LP must be in equality form");
  }
  tol.validate();
  for (size_t i = 1; i < thresholds.size(); ++i) {
    if (!(thresholds[i] < thresholds[i - 1])) {
      throw std::invalid_argument("run_pdhg: thresholds must be strictly decreasing");
    }
  }
  const Index m = std_lp.num_rows(), n = std_lp.num_cols();
  const SparseMat& A = std_lp.A;  // compressed (lp.cpp:71): borrowed zero-copy
  cclp_cu_lp lp{m, n, A.outerIndexPtr(), A.innerIndexPtr(), A.valuePtr(), std_lp.c.data(),
                std_lp.row_lower.data(), std_lp.row_upper.data(), std_lp.col_lower.data(),
                std_lp.col_upper.data()};
  cclp_cu_config cfg;
  cclp_cu_default_config(&cfg);
  cfg.step_scale = config.step_scale;
  cfg.primal_weight = config.primal_weight;
  cfg.restart_factor = config.restart_factor;
  cfg.time_limit = config.time_limit;
  cfg.norm_iterations = config.norm_iterations;
  cfg.scaling_iterations = config.scaling_iterations;
  cfg.max_iterations = config.max_iterations;
  cfg.check_interval = config.check_interval;
  cfg.seed = config.seed;
  cfg.log_interval = config.log != nullptr ? config.log_interval : 0;
  cfg.deterministic = config.deterministic ? 1 : 0;
  cclp_cu_tolerances t{tol.eps_rel, tol.eps_abs, tol.eps_cross, tol.decrement};

  static_assert(sizeof(std::atomic<bool>) == 1 && std::atomic<bool>::is_always_lock_free,
                "the cancel flag is polled as one byte");
  const volatile uint8_t* cancel_byte = reinterpret_cast<const volatile uint8_t*>(cancel);

  Vector x(n), y(m), z(n);
  cclp_cu_result res;
  SinkBridge bridge{&sink, m, n};
  const char* dev_env = std::getenv("CCLP_CU_DEVICE");
  const int device = dev_env ? std::atoi(dev_env) : 0;
  cclp_cu_ctx* ctx = nullptr;
  int rc = cclp_cu_create(&lp, device, &ctx);
  if (rc == CCLP_CU_OK) {
    bridge.ctx = ctx;
    rc = cclp_cu_solve(ctx, &cfg, &t, thresholds.data(), static_cast<int32_t>(thresholds.size()),
                       &sink_trampoline, &bridge, cancel_byte,
                       config.log != nullptr ? &log_trampoline : nullptr, config.log, x.data(),
                       y.data(), z.data(), &res);
    cclp_cu_destroy(ctx);
  }
  if (bridge.error) std::rethrow_exception(bridge.error);
  if (rc == CCLP_CU_EINVAL) throw std::invalid_argument(cclp_cu_last_error());
  if (rc != CCLP_CU_OK) throw std::runtime_error(std::string("cclp_cu: ") + cclp_cu_last_error());

  PdhgResult out;
  out.iterate.x = std::move(x);
  out.iterate.y = std::move(y);
  out.iterate.z = std::move(z);
  out.iterate.k = res.iterations;
  const cclp_cu_report& r = res.report;
  out.report.rp_norm2 = r.rp_norm2;
  out.report.rd_norm2 = r.rd_norm2;
  out.report.rp_inf = r.rp_inf;
  out.report.rd_inf = r.rd_inf;
  out.report.primal_objective = r.primal_objective;
  out.report.dual_objective = r.dual_objective;
  out.report.gap_abs = r.gap_abs;
  out.report.rel_primal = r.rel_primal;
  out.report.rel_dual = r.rel_dual;
  out.report.rel_gap = r.rel_gap;
  out.report.maxresid_rel = r.maxresid_rel;
  out.report.complementarity = r.complementarity;
  out.stop = static_cast<PdhgStopReason>(res.stop);
  out.iterations = res.iterations;
  out.restarts = res.restarts;
  out.seconds = res.seconds;
  out.error_iteration = res.error_iteration;
  return out;
}

}  // namespace cclp
