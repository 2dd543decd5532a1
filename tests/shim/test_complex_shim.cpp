// Complex128 data through the drop-in shim (paper_1604_06043_b200/shim/idrstab_b200.cpp): the
// reference's own C++ types in, mstab::idrstab_solve / mstab_solve on the B200, compared with the
// unmodified reference solve (idrstab.cpp compiled with its entry points renamed ref_*; see
// oracle/Makefile, b200_test_complex_shim). SURVEY.md §8 f4.
#include <gtest/gtest.h>

#include <cmath>
#include <random>
#include <tuple>

#include "mstab/csr.hpp"
#include "mstab/operator.hpp"
#include "mstab/recycle.hpp"
#include "mstab/solvers/idrstab.hpp"

namespace mstab {
SolveResult ref_idrstab_solve(const LinearOperator& a, const Vector& b, const Vector& x0, const SolverConfig& cfg,
                              const RecycleData* recycle, const FetchPolicy* fetch_policy);
}

using namespace mstab;

namespace {

CsrMatrix helmholtz(std::size_t n, Complex shift) {
  std::vector<std::tuple<std::size_t, std::size_t, Complex>> t;
  for (std::size_t i = 0; i < n; ++i) {
    if (i > 0) t.emplace_back(i, i - 1, Complex(-1.0, 0.05));
    t.emplace_back(i, i, Complex(2.0) + shift);
    if (i + 1 < n) t.emplace_back(i, i + 1, Complex(-1.0, -0.05));
  }
  return CsrMatrix::from_triplets(n, n, std::move(t));
}

Vector cvec(std::uint64_t seed, std::size_t n) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  Vector v(n);
  for (Complex& z : v) {
    const double re = u(rng), im = u(rng);
    z = Complex(re, im);
  }
  return v;
}

double relerr(const Vector& a, const Vector& b) {
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num += std::norm(a[i] - b[i]);
    den += std::norm(b[i]);
  }
  return std::sqrt(num / den);
}

double max_abs_diff(const DenseMatrix& a, const DenseMatrix& b) {
  double m = 0.0;
  for (std::size_t i = 0; i < a.data().size(); ++i) m = std::max(m, std::abs(a.data()[i] - b.data()[i]));
  return m;
}

long diff(std::size_t a, std::size_t b) { return static_cast<long>(a) - static_cast<long>(b); }

}  // namespace

TEST(ComplexShim, FreshSolveMatchesReference) {
  const std::size_t n = 900;
  const CsrMatrix m = helmholtz(n, Complex(0.1, 0.3));
  const CsrOperator op(m);
  ASSERT_FALSE(op.is_real());
  const Vector b = cvec(5, n);
  SolverConfig cfg;
  cfg.s = 4;
  cfg.ell = 2;
  cfg.tol = 1e-9;
  cfg.max_mv = 100000;
  cfg.true_residual_each_cycle = true;
  cfg.seed = 13;
  const FetchPolicy pol = FetchPolicy::at_half_tolerance();
  const SolveResult dev = idrstab_solve(op, b, {}, cfg, nullptr, &pol);
  const SolveResult ref = ref_idrstab_solve(op, b, {}, cfg, nullptr, &pol);
  ASSERT_EQ(ref.report.status, SolveStatus::Converged);
  EXPECT_EQ(dev.report.status, SolveStatus::Converged);
  EXPECT_LE(std::labs(diff(dev.report.cycles, ref.report.cycles)), 2);
  EXPECT_LE(relerr(dev.x, ref.x), 1e-6);
  EXPECT_LE(max_abs_diff(dev.final_data.p, ref.final_data.p), 1e-12);
  EXPECT_FALSE(is_real(std::span<const Complex>(dev.final_data.p.data())));
  EXPECT_EQ(dev.final_data.matrix_fingerprint, op.fingerprint());
  EXPECT_EQ(dev.fetched.has_value(), ref.fetched.has_value());
  // the reference's own validate accepts the device hand-off
  EXPECT_LE(validate(dev.handoff(), op).max_deviation, 1e-6);
  // true residual with the reference's SpMV
  Vector r = op.apply(dev.x);
  double rn = 0.0;
  for (std::size_t i = 0; i < n; ++i) rn += std::norm(b[i] - r[i]);
  EXPECT_LE(std::sqrt(rn), 1e-9 * norm2(b));
}

TEST(ComplexShim, RecycledSolveFromTheReferenceHandOff) {
  const std::size_t n = 900;
  const CsrMatrix m = helmholtz(n, Complex(0.1, 0.3));
  const CsrOperator op(m);
  SolverConfig cfg;
  cfg.s = 4;
  cfg.ell = 2;
  cfg.tol = 1e-9;
  cfg.max_mv = 100000;
  cfg.true_residual_each_cycle = true;
  cfg.seed = 13;
  const FetchPolicy pol = FetchPolicy::at_half_tolerance();
  SolveResult ref = ref_idrstab_solve(op, cvec(5, n), {}, cfg, nullptr, &pol);
  for (int i = 0; i < 2; ++i) {
    const RecycleData h = ref.handoff();
    Vector b = ref.x;
    const Vector g = cvec(100 + i, n);
    for (std::size_t t = 0; t < n; ++t) b[t] += 0.2 * g[t];
    const SolveResult dev = mstab_solve(op, b, {}, cfg, h, &pol);
    ref = ref_idrstab_solve(op, b, {}, cfg, &h, &pol);
    ASSERT_EQ(ref.report.status, SolveStatus::Converged);
    EXPECT_EQ(dev.report.status, SolveStatus::Converged);
    EXPECT_LE(std::labs(diff(dev.report.cycles, ref.report.cycles)), 2);
    EXPECT_LE(relerr(dev.x, ref.x), 1e-6);
    EXPECT_EQ(dev.report.h_mv_aux, ref.report.h_mv_aux);
  }
}

TEST(ComplexShim, RealOperatorComplexRightHandSide) {
  const std::size_t n = 500;
  const CsrMatrix m = CsrMatrix::tridiag(-1.0, 2.5, -0.7, n);
  const CsrOperator op(m);
  ASSERT_TRUE(op.is_real());
  const Vector b = cvec(9, n);
  SolverConfig cfg;
  cfg.s = 3;
  cfg.ell = 1;
  cfg.tol = 1e-10;
  cfg.max_mv = 100000;
  cfg.seed = 2;
  const SolveResult dev = idrstab_solve(op, b, {}, cfg, nullptr, nullptr);
  const SolveResult ref = ref_idrstab_solve(op, b, {}, cfg, nullptr, nullptr);
  EXPECT_EQ(dev.report.status, SolveStatus::Converged);
  EXPECT_LE(std::labs(diff(dev.report.cycles, ref.report.cycles)), 2);
  EXPECT_LE(relerr(dev.x, ref.x), 1e-6);
  EXPECT_LE(max_abs_diff(dev.final_data.p, ref.final_data.p), 1e-12);
}
