// O(nnz) standard form for the race. The reference's
// to_standard_form (standard_form.cpp:23-104) rebuilds A from triplets through
// make_sparse (a sort over all nonzeros, kernels.cpp:20-27) although the result
// is just A with one unit column per non-equality row appended on the right.
// A validated A is already canonical (sorted rows, no duplicates, no zeros),
// so the appended CSC is exactly what make_sparse returns; everything else
// (bounds, names, the map) follows the reference line for line. The race
// calls this; tests check it equals the reference's result field by field.
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "cclp/standard_form.hpp"

namespace cclp {
namespace {

// LinearProgram::validate (lp.cpp:49-86) formats a message string for every
// row and column it checks; this scan tests the same conditions without
// allocating and, on the first violation, defers to validate() itself so the
// exception and its text are the reference's.
void validate_lp(const LinearProgram& lp) {
  const Index m = lp.num_rows();
  const Index n = lp.num_cols();
  bool ok = lp.c.size() == n && lp.row_lower.size() == m && lp.row_upper.size() == m &&
            lp.col_lower.size() == n && lp.col_upper.size() == n &&
            static_cast<Index>(lp.sense.size()) == m &&
            (lp.row_names.empty() || static_cast<Index>(lp.row_names.size()) == m) &&
            (lp.col_names.empty() || static_cast<Index>(lp.col_names.size()) == n) && lp.A.isCompressed();
  for (Index j = 0; ok && j < n; ++j) ok = lp.col_lower[j] <= lp.col_upper[j] && !std::isnan(lp.c[j]);
  for (Index i = 0; ok && i < m; ++i) ok = lp.row_lower[i] <= lp.row_upper[i];
  const auto* off = lp.A.outerIndexPtr();
  const auto* rows = lp.A.innerIndexPtr();
  const auto* vals = lp.A.valuePtr();
  for (Index j = 0; ok && j < n; ++j) {
    ok = off[j] <= off[j + 1];
    for (Index p = off[j]; ok && p < off[j + 1]; ++p)
      ok = rows[p] >= 0 && rows[p] < m && (p == off[j] || rows[p] > rows[p - 1]) && vals[p] != 0.0 &&
           !std::isnan(vals[p]);
  }
  if (!ok) lp.validate();
}

}  // namespace

StandardFormMap to_standard_form_direct(const LinearProgram& lp) {
  validate_lp(lp);
  const Index m = lp.num_rows();
  const Index n = lp.num_cols();
  StandardFormMap map;
  map.orig_cols = n;
  map.orig_rows = m;
  map.negated = lp.obj_sense == ObjSense::kMax;
  map.slack_col_of_row.assign(static_cast<size_t>(m), -1);
  Index n_std = n;
  for (Index i = 0; i < m; ++i)
    if (!row_is_equality(lp, i)) map.slack_col_of_row[static_cast<size_t>(i)] = n_std++;

  LinearProgram& s = map.std_lp;
  s.name = lp.name;
  s.objective_name = lp.objective_name;
  s.obj_sense = ObjSense::kMin;
  s.obj_offset = map.negated ? -lp.obj_offset : lp.obj_offset;
  s.c = Vector::Zero(n_std);
  s.c.head(n) = map.negated ? Vector(-lp.c) : lp.c;
  s.col_lower = Vector::Zero(n_std);
  s.col_upper = Vector::Zero(n_std);
  s.col_lower.head(n) = lp.col_lower;
  s.col_upper.head(n) = lp.col_upper;
  s.row_lower = Vector::Zero(m);
  s.row_upper = Vector::Zero(m);
  s.sense.assign(static_cast<size_t>(m), RowSense::kEq);
  s.row_names = lp.row_names;
  s.col_names = lp.col_names;
  if (s.col_names.empty() && n_std > n)
    for (Index j = 0; j < n; ++j) s.col_names.push_back("C" + std::to_string(j));

  for (Index i = 0; i < m; ++i) {
    const Index k = map.slack_col_of_row[static_cast<size_t>(i)];
    const Scalar rl = lp.row_lower[i], ru = lp.row_upper[i];
    if (k < 0) {
      s.row_lower[i] = rl;
      s.row_upper[i] = ru;
      continue;
    }
    if (!is_finite(rl) && !is_finite(ru))
      throw std::invalid_argument("to_standard_form: free row " + std::to_string(i));
    const Scalar b = is_finite(ru) ? ru : rl;
    s.row_lower[i] = b;
    s.row_upper[i] = b;
    s.col_lower[k] = is_finite(ru) ? 0.0 : -kInf;
    s.col_upper[k] = is_finite(rl) ? b - rl : kInf;
    if (!s.col_names.empty())
      s.col_names.push_back("SLK_" + (lp.row_names.empty() ? "R" + std::to_string(i)
                                                             : lp.row_names[static_cast<size_t>(i)]));
  }

  if (n_std == n) {
    s.A = lp.A;
  } else {
    const Index nnz = static_cast<Index>(lp.A.nonZeros());
    const Index extra = n_std - n;
    std::vector<int> colptr(static_cast<size_t>(n_std) + 1), rowind(static_cast<size_t>(nnz + extra));
    std::vector<Scalar> val(static_cast<size_t>(nnz + extra));
    const auto* op = lp.A.outerIndexPtr();
    const auto* ip = lp.A.innerIndexPtr();
    const auto* vp = lp.A.valuePtr();
    for (Index j = 0; j <= n; ++j) colptr[static_cast<size_t>(j)] = static_cast<int>(op[j]);
    for (Index e = 0; e < nnz; ++e) {
      rowind[static_cast<size_t>(e)] = static_cast<int>(ip[e]);
      val[static_cast<size_t>(e)] = vp[e];
    }
    Index e = nnz;
    for (Index i = 0; i < m; ++i) {
      if (map.slack_col_of_row[static_cast<size_t>(i)] < 0) continue;
      rowind[static_cast<size_t>(e)] = static_cast<int>(i);
      val[static_cast<size_t>(e)] = 1.0;
      ++e;
      colptr[static_cast<size_t>(n + (e - nnz))] = static_cast<int>(e);
    }
    s.A = SparseMat(Eigen::Map<SparseMat>(m, n_std, static_cast<int>(nnz + extra), colptr.data(),
                                          rowind.data(), val.data()));
  }
  // The output is valid by construction (a valid A with unit columns
  // appended, b on a finite side); the reference re-validates it, this
  // checks it with the same conditions.
  validate_lp(s);
  return map;
}

}  // namespace cclp
