// Shared by the C ABI's translation units (capi.cu, sharded.cu): the opaque
// context type, error mapping and the run_pdhg preconditions.
#pragma once

#include "context.cuh"

using cclp_cu::Context;
using cclp_cu::Ctrl;
using cclp_cu::Error;
using cclp_cu::g_err;

struct cclp_cu_ctx {
  Context c;
};

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return CCLP_CU_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return CCLP_CU_EINVAL;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    return CCLP_CU_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CCLP_CU_ECUDA;
  }
}

void validate_inputs_eq(bool equality, const cclp_cu_config& cfg, const cclp_cu_tolerances& tol,
                        const double* thr, int nthr) {
  // run_pdhg preconditions (pdhg.cpp:235-244, kkt.cpp:26-37)
  if (!equality) throw std::invalid_argument("run_pdhg: LP must be in equality form");
  if (!(tol.decrement > 0.0 && tol.decrement < 1.0))
    throw std::invalid_argument("tolerances: decrement must be in (0,1)");
  if (!(tol.eps_rel > 0.0 && tol.eps_rel <= tol.eps_cross))
    throw std::invalid_argument("tolerances: need 0 < eps_rel <= eps_cross");
  if (!(tol.eps_abs > 0.0)) throw std::invalid_argument("tolerances: eps_abs must be positive");
  for (int i = 1; i < nthr; ++i)
    if (!(thr[i] < thr[i - 1]))
      throw std::invalid_argument("run_pdhg: thresholds must be strictly decreasing");
  if (cfg.check_interval <= 0)  // modulo by zero in the reference (pdhg.cpp:311)
    throw std::invalid_argument("run_pdhg: check_interval must be positive");
}

void validate_inputs(const cclp_cu_ctx* ctx, const cclp_cu_config& cfg, const cclp_cu_tolerances& tol,
                     const double* thr, int nthr) {
  validate_inputs_eq(ctx->c.equality, cfg, tol, thr, nthr);
}

void copy_report(const double* src, cclp_cu_report* dst) {
  std::memcpy(dst, src, sizeof(double) * cclp_cu::kRepN);
}

}  // namespace
