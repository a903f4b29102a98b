// Eigen-API-subset shim — TEST INFRASTRUCTURE ONLY.
//
// Eigen (>= 3.4, required by the reference at proj/CMakeLists.txt:12) is not
// installed in this image and there is no network. This header implements
// exactly the slice of the Eigen API that the reference's hot-path sources
// (proj/src/{lp,kernels,scaling,kkt,pdhg,standard_form}.cpp) and their tests
// (proj/tests/test_{kernels,scaling,kkt,pdhg,standard_form}.cpp) use, so that
// those files compile UNMODIFIED into oracle/_ref/. It is never linked into
// the product library.
//
// Arithmetic semantics follow Eigen 3.4.0 on x86-64 (SSE2, 2-wide double
// packets, no FMA contraction):
//  * coefficient-wise expressions are lazy expression templates, evaluated per
//    coefficient in the same operation order Eigen uses;
//  * sum/dot/squaredNorm use Eigen's LinearVectorizedTraversal redux: two
//    2-wide packet accumulators over aligned pairs, combined, horizontally
//    added, then the odd tail (Redux.h, redux_impl<..., LinearVectorized...>);
//  * ColMajor sparse * dense is a column scatter res[i] += a_ij * x_j in
//    ascending j (SparseDenseProduct.h, ColMajor branch);
//  * (ColMajor)^T * dense is a per-column gather tmp += a_ij * y_i in
//    ascending i, then res_j += 1 * tmp (RowMajor branch, processRow);
//  * setFromTriplets sums duplicates in insertion order; prune(0,0) removes
//    exact zeros.
#ifndef CCLP_ORACLE_EIGEN_SHIM_H_
#define CCLP_ORACLE_EIGEN_SHIM_H_

#include <algorithm>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <initializer_list>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
enum : int { Dynamic = -1 };
const int Infinity = -1;
enum StorageOptions { ColMajor = 0, RowMajor = 0x1 };
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };

class VectorXd;
class MatrixXd;

namespace internal {

// Eigen 3.4 redux for a linear, vectorizable expression with 2-wide packets.
template <typename F>
inline double redux_sum(Index n, F coeff) {
  if (n == 0) return 0.0;
  const Index ps = 2;
  const Index aligned2 = (n / (2 * ps)) * (2 * ps);
  const Index aligned = (n / ps) * ps;
  double res;
  if (aligned) {
    double p0a = coeff(0), p0b = coeff(1);
    if (aligned > ps) {
      double p1a = coeff(2), p1b = coeff(3);
      for (Index i = 2 * ps; i < aligned2; i += 2 * ps) {
        p0a = p0a + coeff(i);
        p0b = p0b + coeff(i + 1);
        p1a = p1a + coeff(i + 2);
        p1b = p1b + coeff(i + 3);
      }
      p0a = p0a + p1a;
      p0b = p0b + p1b;
      if (aligned > aligned2) {
        p0a = p0a + coeff(aligned2);
        p0b = p0b + coeff(aligned2 + 1);
      }
    }
    res = p0a + p0b;
    for (Index i = aligned; i < n; ++i) res = res + coeff(i);
  } else {
    res = coeff(0);
    for (Index i = 1; i < n; ++i) res = res + coeff(i);
  }
  return res;
}

inline double maxi(double a, double b) { return (a < b) ? b : a; }
inline double mini(double a, double b) { return (b < a) ? b : a; }

}  // namespace internal

// ---------------------------------------------------------------------------
// Dense column-vector expressions.
// ---------------------------------------------------------------------------

template <typename Derived>
class ArrayWrap;
template <typename Derived>
class VecBase;

template <typename T>
struct is_vec_expr {
  template <typename D>
  static std::true_type test(const VecBase<D>*);
  static std::false_type test(...);
  static constexpr bool value =
      decltype(test(std::declval<const std::decay_t<T>*>()))::value;
};

// Leaves (VectorXd) are held by reference; interior nodes by value.
template <typename T>
struct node_storage {
  using type = std::conditional_t<std::is_same<std::decay_t<T>, VectorXd>::value,
                                  const VectorXd&, const std::decay_t<T>>;
};

template <typename Op, typename L, typename R>
class BinaryExpr;
template <typename Op, typename E>
class UnaryExpr;

struct OpAdd { double operator()(double a, double b) const { return a + b; } };
struct OpSub { double operator()(double a, double b) const { return a - b; } };
struct OpMul { double operator()(double a, double b) const { return a * b; } };
struct OpDiv { double operator()(double a, double b) const { return a / b; } };
struct OpMax { double operator()(double a, double b) const { return internal::maxi(a, b); } };
struct OpMin { double operator()(double a, double b) const { return internal::mini(a, b); } };
struct OpNeg { double operator()(double a) const { return -a; } };
struct OpAbs { double operator()(double a) const { return std::abs(a); } };
struct OpAbs2 { double operator()(double a) const { return a * a; } };
struct OpInv { double operator()(double a) const { return 1.0 / a; } };
struct OpScalarMulL { double s; double operator()(double a) const { return s * a; } };
struct OpScalarMulR { double s; double operator()(double a) const { return a * s; } };
struct OpScalarDiv { double s; double operator()(double a) const { return a / s; } };
struct OpScalarMax { double s; double operator()(double a) const { return internal::maxi(a, s); } };
struct OpScalarMin { double s; double operator()(double a) const { return internal::mini(a, s); } };

template <typename Derived>
class VecBase {
 public:
  const Derived& derived() const { return static_cast<const Derived&>(*this); }
  Index size() const { return derived().size(); }
  Index rows() const { return derived().size(); }
  Index cols() const { return 1; }
  double coeff(Index i) const { return derived().coeff(i); }

  template <typename O>
  BinaryExpr<OpMax, Derived, O> cwiseMax(const VecBase<O>& o) const {
    return {derived(), o.derived()};
  }
  template <typename O>
  BinaryExpr<OpMin, Derived, O> cwiseMin(const VecBase<O>& o) const {
    return {derived(), o.derived()};
  }
  UnaryExpr<OpScalarMax, Derived> cwiseMax(double s) const { return {derived(), OpScalarMax{s}}; }
  UnaryExpr<OpScalarMin, Derived> cwiseMin(double s) const { return {derived(), OpScalarMin{s}}; }
  template <typename O>
  BinaryExpr<OpMul, Derived, O> cwiseProduct(const VecBase<O>& o) const {
    return {derived(), o.derived()};
  }
  template <typename O>
  BinaryExpr<OpDiv, Derived, O> cwiseQuotient(const VecBase<O>& o) const {
    return {derived(), o.derived()};
  }
  UnaryExpr<OpInv, Derived> cwiseInverse() const { return {derived(), OpInv{}}; }
  UnaryExpr<OpAbs, Derived> cwiseAbs() const { return {derived(), OpAbs{}}; }
  UnaryExpr<OpAbs2, Derived> cwiseAbs2() const { return {derived(), OpAbs2{}}; }
  UnaryExpr<OpNeg, Derived> operator-() const { return {derived(), OpNeg{}}; }

  double sum() const {
    const Derived& d = derived();
    return internal::redux_sum(d.size(), [&](Index i) { return d.coeff(i); });
  }
  template <typename O>
  double dot(const VecBase<O>& o) const {
    const Derived& a = derived();
    const O& b = o.derived();
    if (a.size() != b.size()) throw std::invalid_argument("Eigen shim: dot size mismatch");
    return internal::redux_sum(a.size(), [&](Index i) { return a.coeff(i) * b.coeff(i); });
  }
  double squaredNorm() const {
    const Derived& d = derived();
    return internal::redux_sum(d.size(), [&](Index i) {
      const double v = d.coeff(i);
      return v * v;
    });
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  double maxCoeff() const {
    const Derived& d = derived();
    assert(d.size() > 0);
    double r = d.coeff(0);
    for (Index i = 1; i < d.size(); ++i) r = internal::maxi(r, d.coeff(i));
    return r;
  }
  double minCoeff() const {
    const Derived& d = derived();
    assert(d.size() > 0);
    double r = d.coeff(0);
    for (Index i = 1; i < d.size(); ++i) r = internal::mini(r, d.coeff(i));
    return r;
  }
  template <int P>
  double lpNorm() const {
    static_assert(P == Infinity, "Eigen shim: only lpNorm<Infinity>");
    const Derived& d = derived();
    if (d.size() == 0) return 0.0;
    double r = std::abs(d.coeff(0));
    for (Index i = 1; i < d.size(); ++i) r = internal::maxi(r, std::abs(d.coeff(i)));
    return r;
  }
  bool allFinite() const {
    const Derived& d = derived();
    for (Index i = 0; i < d.size(); ++i) {
      const double v = d.coeff(i);
      if (std::isnan(v - v)) return false;
    }
    return true;
  }
  bool isZero(double prec = 1e-12) const {
    const Derived& d = derived();
    for (Index i = 0; i < d.size(); ++i)
      if (!(std::abs(d.coeff(i)) <= prec)) return false;
    return true;
  }
  template <typename O>
  bool operator==(const VecBase<O>& o) const {
    const Derived& a = derived();
    const O& b = o.derived();
    assert(a.size() == b.size());
    if (a.size() != b.size()) return false;
    for (Index i = 0; i < a.size(); ++i)
      if (!(a.coeff(i) == b.coeff(i))) return false;
    return true;
  }
  template <typename O>
  bool operator!=(const VecBase<O>& o) const { return !(*this == o); }
  ArrayWrap<Derived> array() const { return ArrayWrap<Derived>(derived()); }
};

template <typename Op, typename L, typename R>
class BinaryExpr : public VecBase<BinaryExpr<Op, L, R>> {
 public:
  BinaryExpr(const L& l, const R& r, Op op = Op{}) : l_(l), r_(r), op_(op) {
    if (l.size() != r.size()) throw std::invalid_argument("Eigen shim: size mismatch");
  }
  Index size() const { return l_.size(); }
  double coeff(Index i) const { return op_(l_.coeff(i), r_.coeff(i)); }
  double operator[](Index i) const { return coeff(i); }

 private:
  typename node_storage<L>::type l_;
  typename node_storage<R>::type r_;
  Op op_;
};

template <typename Op, typename E>
class UnaryExpr : public VecBase<UnaryExpr<Op, E>> {
 public:
  UnaryExpr(const E& e, Op op) : e_(e), op_(op) {}
  Index size() const { return e_.size(); }
  double coeff(Index i) const { return op_(e_.coeff(i)); }
  double operator[](Index i) const { return coeff(i); }

 private:
  typename node_storage<E>::type e_;
  Op op_;
};

template <typename L, typename R>
BinaryExpr<OpAdd, L, R> operator+(const VecBase<L>& l, const VecBase<R>& r) {
  return {l.derived(), r.derived()};
}
template <typename L, typename R>
BinaryExpr<OpSub, L, R> operator-(const VecBase<L>& l, const VecBase<R>& r) {
  return {l.derived(), r.derived()};
}
template <typename E>
UnaryExpr<OpScalarMulL, E> operator*(double s, const VecBase<E>& e) {
  return {e.derived(), OpScalarMulL{s}};
}
template <typename E>
UnaryExpr<OpScalarMulR, E> operator*(const VecBase<E>& e, double s) {
  return {e.derived(), OpScalarMulR{s}};
}
template <typename E>
UnaryExpr<OpScalarDiv, E> operator/(const VecBase<E>& e, double s) {
  return {e.derived(), OpScalarDiv{s}};
}

// Boolean arrays for `(a.array() >= b.array()).all()`.
template <typename F>
class BoolArray {
 public:
  BoolArray(Index n, F f) : n_(n), f_(f) {}
  bool all() const {
    for (Index i = 0; i < n_; ++i)
      if (!f_(i)) return false;
    return true;
  }
  bool any() const {
    for (Index i = 0; i < n_; ++i)
      if (f_(i)) return true;
    return false;
  }
  Index count() const {
    Index c = 0;
    for (Index i = 0; i < n_; ++i) c += f_(i) ? 1 : 0;
    return c;
  }

 private:
  Index n_;
  F f_;
};

template <typename Derived>
class ArrayWrap {
 public:
  explicit ArrayWrap(const Derived& d) : d_(d) {}
  const Derived& vec() const { return d_; }
#define CCLP_SHIM_CMP(OP)                                                        \
  template <typename O>                                                          \
  auto operator OP(const ArrayWrap<O>& o) const {                                \
    const Derived& a = d_;                                                       \
    const O& b = o.vec();                                                        \
    auto f = [&a, &b](Index i) { return a.coeff(i) OP b.coeff(i); };             \
    return BoolArray<decltype(f)>(a.size(), f);                                  \
  }                                                                              \
  auto operator OP(double s) const {                                             \
    const Derived& a = d_;                                                       \
    auto f = [&a, s](Index i) { return a.coeff(i) OP s; };                       \
    return BoolArray<decltype(f)>(a.size(), f);                                  \
  }
  CCLP_SHIM_CMP(>=)
  CCLP_SHIM_CMP(<=)
  CCLP_SHIM_CMP(>)
  CCLP_SHIM_CMP(<)
  CCLP_SHIM_CMP(==)
#undef CCLP_SHIM_CMP
 private:
  const Derived& d_;
};

// Writable contiguous segment of a VectorXd (head/tail/segment).
class VectorBlock : public VecBase<VectorBlock> {
 public:
  VectorBlock(double* p, Index n) : p_(p), n_(n) {}
  Index size() const { return n_; }
  double coeff(Index i) const { return p_[i]; }
  double operator[](Index i) const { return p_[i]; }
  double& operator[](Index i) { return p_[i]; }
  const double* data() const { return p_; }
  template <typename E>
  VectorBlock& operator=(const VecBase<E>& e) {
    const E& d = e.derived();
    if (d.size() != n_) throw std::invalid_argument("Eigen shim: block size mismatch");
    std::vector<double> tmp(n_);
    for (Index i = 0; i < n_; ++i) tmp[i] = d.coeff(i);
    std::copy(tmp.begin(), tmp.end(), p_);
    return *this;
  }
  VectorBlock& operator=(const VectorBlock& o) {
    return operator=(static_cast<const VecBase<VectorBlock>&>(o));
  }
  template <typename E>
  VectorBlock& operator+=(const VecBase<E>& e) {
    const E& d = e.derived();
    for (Index i = 0; i < n_; ++i) p_[i] = p_[i] + d.coeff(i);
    return *this;
  }
  template <typename E>
  VectorBlock& operator-=(const VecBase<E>& e) {
    const E& d = e.derived();
    for (Index i = 0; i < n_; ++i) p_[i] = p_[i] - d.coeff(i);
    return *this;
  }
  VectorBlock& setZero() {
    std::fill(p_, p_ + n_, 0.0);
    return *this;
  }

 private:
  double* p_;
  Index n_;
};

class VectorXd : public VecBase<VectorXd> {
 public:
  using Scalar = double;
  VectorXd() = default;
  explicit VectorXd(Index n) : v_(static_cast<size_t>(n)) {}
  VectorXd(const VectorXd&) = default;
  VectorXd(VectorXd&&) noexcept = default;
  VectorXd& operator=(const VectorXd&) = default;
  VectorXd& operator=(VectorXd&&) noexcept = default;
  template <typename E>
  VectorXd(const VecBase<E>& e) {  // NOLINT: implicit like Eigen
    assign(e.derived());
  }
  template <typename E>
  VectorXd& operator=(const VecBase<E>& e) {
    assign(e.derived());
    return *this;
  }
  // Eigen 3.4: a single inner list on a column vector gives its coefficients.
  VectorXd(std::initializer_list<std::initializer_list<double>> rows) {
    if (rows.size() == 1) {
      v_.assign(rows.begin()->begin(), rows.begin()->end());
    } else {
      for (const auto& r : rows) {
        if (r.size() != 1) throw std::invalid_argument("Eigen shim: bad init list");
        v_.push_back(*r.begin());
      }
    }
  }

  static VectorXd Zero(Index n) { return Constant(n, 0.0); }
  static VectorXd Ones(Index n) { return Constant(n, 1.0); }
  static VectorXd Constant(Index n, double c) {
    VectorXd v(n);
    std::fill(v.v_.begin(), v.v_.end(), c);
    return v;
  }

  Index size() const { return static_cast<Index>(v_.size()); }
  double coeff(Index i) const { return v_[static_cast<size_t>(i)]; }
  double& coeffRef(Index i) { return v_[static_cast<size_t>(i)]; }
  double operator[](Index i) const { return v_[static_cast<size_t>(i)]; }
  double& operator[](Index i) { return v_[static_cast<size_t>(i)]; }
  double operator()(Index i) const { return v_[static_cast<size_t>(i)]; }
  double& operator()(Index i) { return v_[static_cast<size_t>(i)]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  void resize(Index n) { v_.resize(static_cast<size_t>(n)); }
  VectorXd& setZero() { return setConstant(0.0); }
  VectorXd& setOnes() { return setConstant(1.0); }
  VectorXd& setConstant(double c) {
    std::fill(v_.begin(), v_.end(), c);
    return *this;
  }
  VectorXd& setZero(Index n) {
    resize(n);
    return setZero();
  }
  VectorBlock head(Index n) { return VectorBlock(data(), n); }
  VectorBlock tail(Index n) { return VectorBlock(data() + size() - n, n); }
  VectorBlock segment(Index s, Index n) { return VectorBlock(data() + s, n); }
  VectorXd head(Index n) const { return VectorXd(v_.begin(), v_.begin() + n); }
  VectorXd tail(Index n) const { return VectorXd(v_.end() - n, v_.end()); }
  VectorXd segment(Index s, Index n) const {
    return VectorXd(v_.begin() + s, v_.begin() + s + n);
  }

  template <typename E>
  VectorXd& operator+=(const VecBase<E>& e) {
    const E& d = e.derived();
    check(d.size());
    for (Index i = 0; i < size(); ++i) v_[i] = v_[i] + d.coeff(i);
    return *this;
  }
  template <typename E>
  VectorXd& operator-=(const VecBase<E>& e) {
    const E& d = e.derived();
    check(d.size());
    for (Index i = 0; i < size(); ++i) v_[i] = v_[i] - d.coeff(i);
    return *this;
  }
  VectorXd& operator*=(double s) {
    for (auto& x : v_) x = x * s;
    return *this;
  }
  VectorXd& operator/=(double s) {
    for (auto& x : v_) x = x / s;
    return *this;
  }

 private:
  template <typename It>
  VectorXd(It b, It e) : v_(b, e) {}
  void check(Index n) const {
    if (n != size()) throw std::invalid_argument("Eigen shim: size mismatch");
  }
  template <typename E>
  void assign(const E& d) {
    const Index n = d.size();
    std::vector<double> tmp(static_cast<size_t>(n));  // no-alias evaluation
    for (Index i = 0; i < n; ++i) tmp[i] = d.coeff(i);
    v_.swap(tmp);
  }
  std::vector<double> v_;
};

// Map<const VectorXd> / Map<VectorXd>: a view over external storage.
template <typename T>
class Map;
template <>
class Map<const VectorXd> : public VecBase<Map<const VectorXd>> {
 public:
  Map(const double* p, Index n) : p_(p), n_(n) {}
  Index size() const { return n_; }
  double coeff(Index i) const { return p_[i]; }
  double operator[](Index i) const { return p_[i]; }
  const double* data() const { return p_; }

 private:
  const double* p_;
  Index n_;
};

// Ref<const VectorXd>: binds to a vector without copying, or evaluates an
// expression into owned storage (as Eigen does for non-contiguous inputs).
template <typename T>
class Ref;
template <>
class Ref<const VectorXd> : public VecBase<Ref<const VectorXd>> {
 public:
  Ref(const VectorXd& v) : p_(v.data()), n_(v.size()) {}  // NOLINT
  Ref(const VectorBlock& b) : p_(b.data()), n_(b.size()) {}  // NOLINT
  Ref(const Map<const VectorXd>& m) : p_(m.data()), n_(m.size()) {}  // NOLINT
  template <typename E,
            typename = std::enable_if_t<!std::is_same<E, VectorXd>::value &&
                                        !std::is_same<E, VectorBlock>::value>>
  Ref(const VecBase<E>& e) : own_(e), p_(own_.data()), n_(own_.size()) {}  // NOLINT
  Ref(const Ref& o) : own_(o.own_), p_(o.p_), n_(o.n_) {
    if (o.p_ == o.own_.data()) p_ = own_.data();
  }
  Index size() const { return n_; }
  double coeff(Index i) const { return p_[i]; }
  double operator[](Index i) const { return p_[i]; }
  const double* data() const { return p_; }
  Map<const VectorXd> head(Index n) const { return Map<const VectorXd>(p_, n); }
  Map<const VectorXd> tail(Index n) const { return Map<const VectorXd>(p_ + n_ - n, n); }
  Map<const VectorXd> segment(Index s, Index n) const { return Map<const VectorXd>(p_ + s, n); }

 private:
  VectorXd own_;
  const double* p_;
  Index n_;
};

// ---------------------------------------------------------------------------
// Sparse matrices (compressed column-major only).
// ---------------------------------------------------------------------------

template <typename S = double, typename I = int>
class Triplet {
 public:
  Triplet() : r_(0), c_(0), v_(0) {}
  Triplet(const I& r, const I& c, const S& v = S(0)) : r_(r), c_(c), v_(v) {}
  const I& row() const { return r_; }
  const I& col() const { return c_; }
  const S& value() const { return v_; }

 private:
  I r_, c_;
  S v_;
};

template <typename S, int Options = ColMajor, typename I = int>
class SparseMatrix;

template <typename S, int O, typename I>
class Map<SparseMatrix<S, O, I>> {
 public:
  Map(Index rows, Index cols, Index nnz, const I* outer, const I* inner, const S* vals)
      : rows_(rows), cols_(cols), nnz_(nnz), outer_(outer), inner_(inner), vals_(vals) {}
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index nonZeros() const { return nnz_; }
  const I* outerIndexPtr() const { return outer_; }
  const I* innerIndexPtr() const { return inner_; }
  const S* valuePtr() const { return vals_; }

 private:
  Index rows_, cols_, nnz_;
  const I* outer_;
  const I* inner_;
  const S* vals_;
};

template <typename M>
class SparseTransposeView;
template <typename M>
class SparseLeftColsView;

template <typename S, int Options, typename I>
class SparseMatrix {
  static_assert(std::is_same<S, double>::value, "Eigen shim: double only");
  static_assert(Options == ColMajor, "Eigen shim: ColMajor only");

 public:
  using Scalar = S;
  using StorageIndex = I;

  SparseMatrix() : rows_(0), cols_(0), outer_(1, 0) {}
  SparseMatrix(Index r, Index c) : rows_(r), cols_(c), outer_(static_cast<size_t>(c) + 1, 0) {}
  SparseMatrix(const Map<SparseMatrix>& m)  // NOLINT: implicit like Eigen
      : rows_(m.rows()),
        cols_(m.cols()),
        outer_(m.outerIndexPtr(), m.outerIndexPtr() + m.cols() + 1),
        inner_(m.innerIndexPtr(), m.innerIndexPtr() + m.nonZeros()),
        vals_(m.valuePtr(), m.valuePtr() + m.nonZeros()) {}

  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index outerSize() const { return cols_; }
  Index innerSize() const { return rows_; }
  Index nonZeros() const { return static_cast<Index>(vals_.size()); }
  bool isCompressed() const { return true; }
  void makeCompressed() {}
  void resize(Index r, Index c) {
    rows_ = r;
    cols_ = c;
    outer_.assign(static_cast<size_t>(c) + 1, 0);
    inner_.clear();
    vals_.clear();
  }
  void setZero() {
    inner_.clear();
    vals_.clear();
    std::fill(outer_.begin(), outer_.end(), 0);
  }
  void reserve(Index nnz) {
    inner_.reserve(static_cast<size_t>(nnz));
    vals_.reserve(static_cast<size_t>(nnz));
  }
  const I* outerIndexPtr() const { return outer_.data(); }
  const I* innerIndexPtr() const { return inner_.data(); }
  const S* valuePtr() const { return vals_.data(); }
  I* outerIndexPtr() { return outer_.data(); }
  I* innerIndexPtr() { return inner_.data(); }
  S* valuePtr() { return vals_.data(); }
  const I* innerNonZeroPtr() const { return nullptr; }

  template <typename It>
  void setFromTriplets(It begin, It end) {
    std::vector<Triplet<S, I>> t;
    for (It it = begin; it != end; ++it) t.emplace_back(it->row(), it->col(), it->value());
    std::vector<size_t> order(t.size());
    std::iota(order.begin(), order.end(), size_t{0});
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
      if (t[a].col() != t[b].col()) return t[a].col() < t[b].col();
      return t[a].row() < t[b].row();
    });
    inner_.clear();
    vals_.clear();
    std::fill(outer_.begin(), outer_.end(), 0);
    I last_r = -1, last_c = -1;
    for (size_t k : order) {
      const auto& e = t[k];
      if (e.row() < 0 || e.row() >= rows_ || e.col() < 0 || e.col() >= cols_)
        throw std::invalid_argument("Eigen shim: triplet out of range");
      if (e.row() == last_r && e.col() == last_c) {
        vals_.back() = vals_.back() + e.value();
      } else {
        inner_.push_back(e.row());
        vals_.push_back(e.value());
        outer_[static_cast<size_t>(e.col()) + 1]++;
        last_r = e.row();
        last_c = e.col();
      }
    }
    for (Index j = 0; j < cols_; ++j) outer_[j + 1] += outer_[j];
  }

  void prune(const S& reference, const double& epsilon) {
    I w = 0;
    I start = 0;
    for (Index j = 0; j < cols_; ++j) {
      const I end = outer_[j + 1];
      for (I p = start; p < end; ++p) {
        if (!(std::abs(vals_[p]) <= std::abs(reference) * epsilon)) {
          inner_[w] = inner_[p];
          vals_[w] = vals_[p];
          ++w;
        }
      }
      start = end;
      outer_[j + 1] = w;
    }
    inner_.resize(w);
    vals_.resize(w);
  }

  S coeff(Index r, Index c) const {
    const I* b = inner_.data() + outer_[c];
    const I* e = inner_.data() + outer_[c + 1];
    const I* p = std::lower_bound(b, e, static_cast<I>(r));
    return (p != e && *p == r) ? vals_[p - inner_.data()] : S(0);
  }
  S& coeffRef(Index r, Index c) {
    const size_t b = outer_[c], e = outer_[c + 1];
    auto it = std::lower_bound(inner_.begin() + b, inner_.begin() + e, static_cast<I>(r));
    const size_t pos = static_cast<size_t>(it - inner_.begin());
    if (pos < e && inner_[pos] == r) return vals_[pos];
    inner_.insert(inner_.begin() + pos, static_cast<I>(r));
    vals_.insert(vals_.begin() + pos, S(0));
    for (Index j = c + 1; j <= cols_; ++j) outer_[j]++;
    return vals_[pos];
  }
  S& insert(Index r, Index c) { return coeffRef(r, c); }

  class InnerIterator {
   public:
    InnerIterator(const SparseMatrix& m, Index outer)
        : m_(const_cast<SparseMatrix*>(&m)), p_(m.outer_[outer]), end_(m.outer_[outer + 1]), outer_(outer) {}
    explicit operator bool() const { return p_ < end_; }
    InnerIterator& operator++() {
      ++p_;
      return *this;
    }
    S value() const { return m_->vals_[p_]; }
    S& valueRef() { return m_->vals_[p_]; }
    I index() const { return m_->inner_[p_]; }
    I row() const { return m_->inner_[p_]; }
    I col() const { return static_cast<I>(outer_); }
    Index outer() const { return outer_; }

   private:
    SparseMatrix* m_;
    I p_, end_;
    Index outer_;
  };

  SparseTransposeView<SparseMatrix> transpose() const { return SparseTransposeView<SparseMatrix>(*this); }
  SparseLeftColsView<SparseMatrix> leftCols(Index k) const { return SparseLeftColsView<SparseMatrix>(*this, k); }

  // ColMajor sparse * dense: scatter in ascending column order.
  template <typename E>
  VectorXd times(const VecBase<E>& xe, Index ncols) const {
    const E& x = xe.derived();
    if (x.size() != ncols) throw std::invalid_argument("Eigen shim: product size mismatch");
    VectorXd res = VectorXd::Zero(rows_);
    double* r = res.data();
    for (Index j = 0; j < ncols; ++j) {
      const double xj = 1.0 * x.coeff(j);
      for (I p = outer_[j]; p < outer_[j + 1]; ++p) r[inner_[p]] += vals_[p] * xj;
    }
    return res;
  }
  template <typename E>
  VectorXd transpose_times(const VecBase<E>& ye) const {
    const E& y = ye.derived();
    if (y.size() != rows_) throw std::invalid_argument("Eigen shim: product size mismatch");
    VectorXd res = VectorXd::Zero(cols_);
    double* r = res.data();
    for (Index j = 0; j < cols_; ++j) {
      double tmp = 0.0;
      for (I p = outer_[j]; p < outer_[j + 1]; ++p) tmp += vals_[p] * y.coeff(inner_[p]);
      r[j] += 1.0 * tmp;
    }
    return res;
  }

 private:
  Index rows_, cols_;
  std::vector<I> outer_;
  std::vector<I> inner_;
  std::vector<S> vals_;
};

template <typename M>
class SparseTransposeView {
 public:
  explicit SparseTransposeView(const M& m) : m_(m) {}
  const M& nested() const { return m_; }
  Index rows() const { return m_.cols(); }
  Index cols() const { return m_.rows(); }

 private:
  const M& m_;
};

template <typename M>
class SparseLeftColsView {
 public:
  SparseLeftColsView(const M& m, Index k) : m_(m), k_(k) {}
  const M& nested() const { return m_; }
  Index cols() const { return k_; }

 private:
  const M& m_;
  Index k_;
};

template <typename S, int O, typename I, typename E>
VectorXd operator*(const SparseMatrix<S, O, I>& A, const VecBase<E>& x) {
  return A.times(x, A.cols());
}
template <typename M, typename E>
VectorXd operator*(const SparseTransposeView<M>& At, const VecBase<E>& y) {
  return At.nested().transpose_times(y);
}
template <typename M, typename E>
VectorXd operator*(const SparseLeftColsView<M>& Ak, const VecBase<E>& x) {
  return Ak.nested().times(x, Ak.cols());
}

using SparseMatrixXd = SparseMatrix<double, ColMajor, int>;

// ---------------------------------------------------------------------------
// Dense matrices (tests only: oracles built from small dense algebra).
// ---------------------------------------------------------------------------

class MatrixXd;

class PartialLU;

class MatrixColumn : public VecBase<MatrixColumn> {
 public:
  MatrixColumn(double* p, Index n) : p_(p), n_(n) {}
  Index size() const { return n_; }
  double coeff(Index i) const { return p_[i]; }
  double operator[](Index i) const { return p_[i]; }
  template <typename E>
  MatrixColumn& operator=(const VecBase<E>& e) {
    const E& d = e.derived();
    std::vector<double> tmp(n_);
    for (Index i = 0; i < n_; ++i) tmp[i] = d.coeff(i);
    std::copy(tmp.begin(), tmp.end(), p_);
    return *this;
  }
  MatrixColumn& operator=(const MatrixColumn& o) {
    return operator=(static_cast<const VecBase<MatrixColumn>&>(o));
  }

 private:
  double* p_;
  Index n_;
};

class MatrixXd {
 public:
  MatrixXd() : r_(0), c_(0) {}
  MatrixXd(Index r, Index c) : r_(r), c_(c), d_(static_cast<size_t>(r * c), 0.0) {}
  template <typename S, int O, typename I>
  explicit MatrixXd(const SparseMatrix<S, O, I>& A) : MatrixXd(A.rows(), A.cols()) {
    for (Index j = 0; j < A.cols(); ++j)
      for (typename SparseMatrix<S, O, I>::InnerIterator it(A, j); it; ++it) (*this)(it.row(), j) = it.value();
  }
  static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }
  static MatrixXd Identity(Index r, Index c) {
    MatrixXd m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  double operator()(Index i, Index j) const { return d_[static_cast<size_t>(j * r_ + i)]; }
  double& operator()(Index i, Index j) { return d_[static_cast<size_t>(j * r_ + i)]; }
  double coeff(Index i, Index j) const { return (*this)(i, j); }
  MatrixColumn col(Index j) { return MatrixColumn(d_.data() + j * r_, r_); }
  MatrixColumn col(Index j) const { return MatrixColumn(const_cast<double*>(d_.data()) + j * r_, r_); }
  MatrixXd transpose() const {
    MatrixXd t(c_, r_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  MatrixXd cwiseAbs() const {
    MatrixXd t(*this);
    for (auto& v : t.d_) v = std::abs(v);
    return t;
  }
  PartialLU lu() const;
  double maxCoeff() const {
    if (d_.empty()) throw std::invalid_argument("Eigen shim: maxCoeff of an empty matrix");
    double mx = d_[0];
    for (double v : d_) mx = (mx < v) ? v : mx;
    return mx;
  }
  // row(i) and row(i).tail(k): strided views (factorization.cpp:50-51)
  class RowView : public VecBase<RowView> {
   public:
    RowView(double* p, Index stride, Index n) : p_(p), s_(stride), n_(n) {}
    Index size() const { return n_; }
    double coeff(Index i) const { return p_[i * s_]; }
    double operator[](Index i) const { return p_[i * s_]; }
    RowView tail(Index k) const { return RowView(p_ + (n_ - k) * s_, s_, k); }
    RowView head(Index k) const { return RowView(p_, s_, k); }
    template <typename E>
    RowView& operator-=(const VecBase<E>& e) {
      const E& d = e.derived();
      std::vector<double> tmp(static_cast<size_t>(n_));
      for (Index i = 0; i < n_; ++i) tmp[i] = d.coeff(i);
      for (Index i = 0; i < n_; ++i) p_[i * s_] = p_[i * s_] - tmp[i];
      return *this;
    }
    template <typename E>
    RowView& operator=(const VecBase<E>& e) {
      const E& d = e.derived();
      std::vector<double> tmp(static_cast<size_t>(n_));
      for (Index i = 0; i < n_; ++i) tmp[i] = d.coeff(i);
      for (Index i = 0; i < n_; ++i) p_[i * s_] = tmp[i];
      return *this;
    }

   private:
    double* p_;
    Index s_, n_;
  };
  RowView row(Index i) { return RowView(d_.data() + i, r_, c_); }
  RowView row(Index i) const { return RowView(const_cast<double*>(d_.data()) + i, r_, c_); }
  struct Rowwise {
    const MatrixXd& m;
    VectorXd sum() const {
      VectorXd s = VectorXd::Zero(m.rows());
      for (Index j = 0; j < m.cols(); ++j)
        for (Index i = 0; i < m.rows(); ++i) s[i] += m(i, j);
      return s;
    }
  };
  Rowwise rowwise() const { return Rowwise{*this}; }
  bool operator==(const MatrixXd& o) const { return r_ == o.r_ && c_ == o.c_ && d_ == o.d_; }
  bool operator!=(const MatrixXd& o) const { return !(*this == o); }

 private:
  Index r_, c_;
  std::vector<double> d_;
};

// MatrixXd::lu(): partial-pivoting LU with solve (test_simplex.cpp:62-64).
class PartialLU {
 public:
  explicit PartialLU(const MatrixXd& A) : n_(A.rows()), a_(A), p_(static_cast<size_t>(A.rows())) {
    for (Index i = 0; i < n_; ++i) p_[i] = i;
    for (Index k = 0; k < n_; ++k) {
      Index piv = k;
      for (Index i = k + 1; i < n_; ++i)
        if (std::abs(a_(i, k)) > std::abs(a_(piv, k))) piv = i;
      if (piv != k) {
        for (Index j = 0; j < n_; ++j) std::swap(a_(k, j), a_(piv, j));
        std::swap(p_[k], p_[piv]);
      }
      for (Index i = k + 1; i < n_; ++i) {
        if (a_(k, k) == 0.0) break;
        a_(i, k) /= a_(k, k);
        for (Index j = k + 1; j < n_; ++j) a_(i, j) -= a_(i, k) * a_(k, j);
      }
    }
  }
  template <typename E>
  VectorXd solve(const VecBase<E>& be) const {
    const E& b = be.derived();
    VectorXd x(n_);
    for (Index i = 0; i < n_; ++i) x[i] = b.coeff(p_[i]);
    for (Index i = 0; i < n_; ++i)
      for (Index j = 0; j < i; ++j) x[i] -= a_(i, j) * x[j];
    for (Index i = n_ - 1; i >= 0; --i) {
      for (Index j = i + 1; j < n_; ++j) x[i] -= a_(i, j) * x[j];
      x[i] /= a_(i, i);
    }
    return x;
  }

 private:
  Index n_;
  MatrixXd a_;
  std::vector<Index> p_;
};

inline PartialLU MatrixXd::lu() const { return PartialLU(*this); }

template <typename E>
VectorXd operator*(const MatrixXd& M, const VecBase<E>& xe) {
  const E& x = xe.derived();
  if (x.size() != M.cols()) throw std::invalid_argument("Eigen shim: gemv size mismatch");
  VectorXd r = VectorXd::Zero(M.rows());
  for (Index j = 0; j < M.cols(); ++j) {
    const double xj = x.coeff(j);
    for (Index i = 0; i < M.rows(); ++i) r[i] += M(i, j) * xj;
  }
  return r;
}

// Full-pivoting LU (rank threshold as in Eigen: eps * max(rows, cols) * maxpivot).
template <typename M>
class FullPivLU;
template <>
class FullPivLU<MatrixXd> {
 public:
  explicit FullPivLU(const MatrixXd& A) : lu_(A), n_(A.rows()), rank_(0) {
    if (A.rows() != A.cols()) throw std::invalid_argument("Eigen shim: FullPivLU square only");
    pr_.resize(n_);
    pc_.resize(n_);
    std::iota(pr_.begin(), pr_.end(), Index{0});
    std::iota(pc_.begin(), pc_.end(), Index{0});
    double maxpivot = 0.0;
    std::vector<double> pivots;
    for (Index k = 0; k < n_; ++k) {
      Index bi = k, bj = k;
      double best = -1.0;
      for (Index j = k; j < n_; ++j)
        for (Index i = k; i < n_; ++i)
          if (std::abs(lu_(i, j)) > best) {
            best = std::abs(lu_(i, j));
            bi = i;
            bj = j;
          }
      if (best == 0.0) break;
      if (k == 0) maxpivot = best;
      pivots.push_back(best);
      if (bi != k) {
        for (Index j = 0; j < n_; ++j) std::swap(lu_(k, j), lu_(bi, j));
        std::swap(pr_[k], pr_[bi]);
        ++swaps_;
      }
      if (bj != k) {
        for (Index i = 0; i < n_; ++i) std::swap(lu_(i, k), lu_(i, bj));
        std::swap(pc_[k], pc_[bj]);
        ++swaps_;
      }
      for (Index i = k + 1; i < n_; ++i) {
        lu_(i, k) /= lu_(k, k);
        for (Index j = k + 1; j < n_; ++j) lu_(i, j) -= lu_(i, k) * lu_(k, j);
      }
    }
    const double thr = std::numeric_limits<double>::epsilon() * static_cast<double>(n_);
    for (double p : pivots)
      if (p > thr * maxpivot) ++rank_;
  }
  bool isInvertible() const { return rank_ == n_; }
  double determinant() const {
    if (rank_ < n_ && static_cast<Index>(0) < n_) {
      double d = 1.0;
      for (Index i = 0; i < n_; ++i) d *= lu_(i, i);
      return (swaps_ % 2 ? -d : d);
    }
    double d = 1.0;
    for (Index i = 0; i < n_; ++i) d *= lu_(i, i);
    return (swaps_ % 2 ? -d : d);
  }
  Index rank() const { return rank_; }
  template <typename E>
  VectorXd solve(const VecBase<E>& be) const {
    const E& b = be.derived();
    std::vector<double> y(n_);
    for (Index i = 0; i < n_; ++i) y[i] = b.coeff(pr_[i]);
    for (Index i = 0; i < n_; ++i)
      for (Index k = 0; k < i; ++k) y[i] -= lu_(i, k) * y[k];
    for (Index i = n_ - 1; i >= 0; --i) {
      for (Index k = i + 1; k < n_; ++k) y[i] -= lu_(i, k) * y[k];
      y[i] /= lu_(i, i);
    }
    VectorXd x(n_);
    for (Index i = 0; i < n_; ++i) x[pc_[i]] = y[i];
    return x;
  }

 private:
  int swaps_ = 0;
  MatrixXd lu_;
  Index n_;
  Index rank_;
  std::vector<Index> pr_, pc_;
};

// Singular values via cyclic Jacobi on the Gram matrix (small matrices only).
template <typename M>
class JacobiSVD;
template <>
class JacobiSVD<MatrixXd> {
 public:
  explicit JacobiSVD(const MatrixXd& A) {
    const bool tall = A.rows() >= A.cols();
    const Index k = tall ? A.cols() : A.rows();
    MatrixXd G(k, k);
    for (Index a = 0; a < k; ++a)
      for (Index b = 0; b < k; ++b) {
        double s = 0.0;
        if (tall)
          for (Index i = 0; i < A.rows(); ++i) s += A(i, a) * A(i, b);
        else
          for (Index j = 0; j < A.cols(); ++j) s += A(a, j) * A(b, j);
        G(a, b) = s;
      }
    for (int sweep = 0; sweep < 100; ++sweep) {
      double off = 0.0;
      for (Index p = 0; p < k; ++p)
        for (Index q = p + 1; q < k; ++q) off += G(p, q) * G(p, q);
      if (off < 1e-30) break;
      for (Index p = 0; p < k; ++p)
        for (Index q = p + 1; q < k; ++q) {
          if (G(p, q) == 0.0) continue;
          const double theta = (G(q, q) - G(p, p)) / (2.0 * G(p, q));
          const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
          const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
          for (Index r = 0; r < k; ++r) {
            const double gp = G(r, p), gq = G(r, q);
            G(r, p) = c * gp - s * gq;
            G(r, q) = s * gp + c * gq;
          }
          for (Index r = 0; r < k; ++r) {
            const double gp = G(p, r), gq = G(q, r);
            G(p, r) = c * gp - s * gq;
            G(q, r) = s * gp + c * gq;
          }
        }
    }
    sv_ = VectorXd(k);
    for (Index i = 0; i < k; ++i) sv_[i] = std::sqrt(std::max(G(i, i), 0.0));
    std::sort(sv_.data(), sv_.data() + k, [](double a, double b) { return a > b; });
  }
  const VectorXd& singularValues() const { return sv_; }

 private:
  VectorXd sv_;
};

}  // namespace Eigen

#endif  // CCLP_ORACLE_EIGEN_SHIM_H_
