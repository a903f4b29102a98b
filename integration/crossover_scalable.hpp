// Crossover that scales past the reference's m ~ 1e4.
//
// Same algorithm and interface as the reference's run_crossover
// (crossover.hpp:61-85, crossover.cpp:247-285): guess_partition -> crash
// basis -> two-phase bounded primal simplex cleanup -> verify_basic_optimal.
// What changes is the linear algebra and the pricing:
//  * the crash (build_basis, crossover.cpp:101-150) keeps one dense eta per
//    accepted candidate (O(m^2) memory, O(m^3) time); here it is the
//    equivalent left-looking sparse LU of the accepted candidates, with the
//    reference's own acceptance rule (pivot = the largest replaceable |w_p|,
//    lowest position on ties; reject below 1e-7 max(1, ||w||_inf));
//  * the simplex's basis factorization (factorization.cpp:58-139: SparseLU +
//    dense eta vectors, dense m x m dependent_positions on a singular basis)
//    is a rank-revealing sparse LU with sparse eta vectors; a singular basis
//    is repaired from the unpivoted rows without a dense matrix;
//  * pricing (simplex.cpp:264-296, one A'y per pivot over n + m columns) runs
//    on the B200 through cclp_cu_price when a device pricer is supplied (the
//    reference's price() pick, bit for bit), else on the host.
#pragma once

#include <memory>
#include <mutex>

#include "cclp/crossover.hpp"

struct cclp_cu_ctx;

namespace cclp_xo {

// A device context over the equality-form LP used only for pricing; shared
// by the crossover workers (calls serialized).
class DevicePricer {
 public:
  DevicePricer(const cclp::LinearProgram& std_lp, int device);
  ~DevicePricer();
  DevicePricer(const DevicePricer&) = delete;
  DevicePricer& operator=(const DevicePricer&) = delete;
  // The reference's price() pick (simplex.cpp:264-296); status[n + m] in
  // ColStatus chars, skip[n + m] or null.
  void price(const double* y, const char* status, const unsigned char* skip, bool phase1, double dtol, bool bland,
             long long* entering, int* direction, double* violation);
  long long calls() const { return calls_; }

 private:
  cclp_cu_ctx* ctx_ = nullptr;
  std::mutex mu_;
  long long calls_ = 0;
};

struct ScalableStats {
  long long crash_candidates = 0, crash_accepted = 0;
  long long lu_nnz = 0;  // L + U of the last factorization
  long long device_prices = 0, host_prices = 0;
  double crash_s = 0, simplex_s = 0, verify_s = 0;
};

// run_crossover with the scalable factorization; `pricer` may be null (host
// pricing). Thread-safe for concurrent workers sharing one pricer.
cclp::CrossoverResult run_crossover(const cclp::CrossoverTask& task, DevicePricer* pricer,
                                    ScalableStats* stats = nullptr);

// The crash alone (build_basis semantics), for tests against the reference.
cclp::Basis build_basis(const cclp::LinearProgram& std_lp, const cclp::Partition& partition,
                        ScalableStats* stats = nullptr);

}  // namespace cclp_xo
