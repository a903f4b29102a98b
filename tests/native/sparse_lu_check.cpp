// Checks third_party/eigen_subset's SparseLU (the product crossover's basis
// factorization): residuals of solve / adjoint().solve on random sparse,
// network-like and banded matrices; singular matrices report NumericalIssue;
// factor fill stays sparse on a transportation-style basis.
#include <cstdio>
#include <random>

#include "Eigen/SparseLU"

using SpMat = Eigen::SparseMatrix<double, Eigen::ColMajor, int>;

static double resid(const SpMat& A, const Eigen::VectorXd& x, const Eigen::VectorXd& b, bool tr) {
  Eigen::VectorXd r = tr ? Eigen::VectorXd(A.transpose() * x) : Eigen::VectorXd(A * x);
  double m = 0.0;
  for (Eigen::Index i = 0; i < b.size(); ++i) m = std::max(m, std::abs(r[i] - b[i]));
  return m;
}

static SpMat build(int n, std::vector<Eigen::Triplet<double, int>>& t) {
  SpMat A(n, n);
  A.setFromTriplets(t.begin(), t.end());
  A.makeCompressed();
  return A;
}

int main() {
  int fails = 0;
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> U(-2.0, 2.0);
  for (int kind = 0; kind < 3; ++kind) {
    for (int n : {1, 5, 60, 400, 3000}) {
      std::vector<Eigen::Triplet<double, int>> t;
      for (int j = 0; j < n; ++j) {
        t.emplace_back((j * 7) % n, j, 2.5 + std::abs(U(g)));  // a permuted diagonal
        if (kind == 0)
          for (int k = 0; k < 3; ++k) t.emplace_back(static_cast<int>(g() % n), j, U(g));
        if (kind == 1 && j + 1 < n) t.emplace_back((j * 7 + 7) % n, j, -1.0);  // network-like
        if (kind == 2)
          for (int d = 1; d <= 4 && j + d < n; ++d) t.emplace_back(j + d, j, U(g) * 0.3);  // band
      }
      SpMat A = build(n, t);
      Eigen::SparseLU<SpMat, Eigen::COLAMDOrdering<int>> lu;
      lu.compute(A);
      if (lu.info() != Eigen::Success) {
        std::printf("FAIL kind %d n %d: not factored\n", kind, n);
        ++fails;
        continue;
      }
      Eigen::VectorXd b(n);
      for (int i = 0; i < n; ++i) b[i] = U(g);
      const double r1 = resid(A, lu.solve(b), b, false);
      const double r2 = resid(A, lu.adjoint().solve(b), b, true);
      const bool ok = r1 < 1e-9 && r2 < 1e-9;
      if (!ok) ++fails;
      std::printf("%s kind %d n %d resid %.2e %.2e nnz(A) %ld L %ld U %ld\n", ok ? "ok" : "FAIL", kind, n,
                  r1, r2, static_cast<long>(A.nonZeros()), static_cast<long>(lu.nnzL()),
                  static_cast<long>(lu.nnzU()));
    }
  }
  {  // singular: duplicate column, and a dependent combination
    std::vector<Eigen::Triplet<double, int>> t = {{0, 0, 1.0}, {1, 0, 2.0}, {0, 1, 1.0}, {1, 1, 2.0},
                                                  {2, 2, 1.0}};
    SpMat A = build(3, t);
    Eigen::SparseLU<SpMat, Eigen::COLAMDOrdering<int>> lu;
    lu.compute(A);
    const bool ok = lu.info() != Eigen::Success;
    std::printf("%s singular detected\n", ok ? "ok" : "FAIL");
    if (!ok) ++fails;
  }
  {  // transportation basis (spanning tree of a bipartite graph): fill stays O(n)
    const int S = 300, D = 700, n = S + D;
    std::vector<Eigen::Triplet<double, int>> t;
    int col = 0;
    for (int d = 0; d < D; ++d, ++col) {  // sink d served by source d % S
      t.emplace_back(d % S, col, 1.0);
      t.emplace_back(S + d, col, 1.0);
    }
    for (int s = 0; s + 1 < S; ++s, ++col) {  // link sources through sink s
      t.emplace_back(s + 1, col, 1.0);
      t.emplace_back(S + s, col, 1.0);
    }
    t.emplace_back(0, col, 1.0);  // one slack
    SpMat A = build(n, t);
    Eigen::SparseLU<SpMat, Eigen::COLAMDOrdering<int>> lu;
    lu.compute(A);
    Eigen::VectorXd b(n);
    for (int i = 0; i < n; ++i) b[i] = U(g);
    const bool fact = lu.info() == Eigen::Success;
    const double r = fact ? resid(A, lu.solve(b), b, false) : 1.0;
    const bool ok = fact && r < 1e-9 && lu.nnzL() + lu.nnzU() <= 4 * A.nonZeros();
    std::printf("%s transport basis n %d resid %.2e L %ld U %ld\n", ok ? "ok" : "FAIL", n, r,
                static_cast<long>(lu.nnzL()), static_cast<long>(lu.nnzU()));
    if (!ok) ++fails;
  }
  std::printf("%s\n", fails ? "FAILED" : "ALL OK");
  return fails ? 1 : 0;
}
