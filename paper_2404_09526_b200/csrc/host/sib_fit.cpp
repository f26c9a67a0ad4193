// Measured-SIB fitting (sib_fit.hpp).
#include "sib_fit.hpp"

#include <algorithm>
#include <cmath>
#include <vector>

#include "errors.hpp"

namespace esp {

namespace {

constexpr double kRankTolerance = 1e-9;  // cost_model.cpp:31

// min ||A x - y|| over the active columns of the (n x 3, column-major) design;
// inactive coefficients stay 0. Householder QR with column pivoting; the rank
// counts pivots above kRankTolerance x the largest (Eigen's ColPivHouseholderQR
// threshold rule, as solve_active configures it).
std::array<double, 3> solve_active(const std::vector<double>& design, const std::vector<double>& y,
                                   size_t n, const std::vector<int>& active) {
  const size_t m = active.size();
  std::vector<double> a(n * m);  // column-major sub-design
  for (size_t c = 0; c < m; ++c) {
    std::copy_n(design.begin() + static_cast<std::ptrdiff_t>(active[c] * n), n,
                a.begin() + static_cast<std::ptrdiff_t>(c * n));
  }
  std::vector<double> b = y;
  std::vector<size_t> perm(m);
  for (size_t c = 0; c < m; ++c) perm[c] = c;
  std::vector<double> rdiag(m, 0.0);
  double max_pivot = 0.0;
  size_t rank = 0;
  for (size_t k = 0; k < m && k < n; ++k) {
    // pivot: the remaining column with the largest norm below row k
    size_t best = k;
    double best_norm = -1.0;
    for (size_t c = k; c < m; ++c) {
      double s = 0;
      for (size_t i = k; i < n; ++i) s += a[c * n + i] * a[c * n + i];
      if (s > best_norm) {
        best_norm = s;
        best = c;
      }
    }
    if (best != k) {
      for (size_t i = 0; i < n; ++i) std::swap(a[k * n + i], a[best * n + i]);
      std::swap(perm[k], perm[best]);
    }
    const double norm = std::sqrt(best_norm);
    if (k == 0) max_pivot = norm;
    if (norm <= kRankTolerance * max_pivot || norm == 0.0) break;
    // Householder reflector zeroing column k below the diagonal
    const double alpha = a[k * n + k] > 0 ? -norm : norm;
    std::vector<double> v(n, 0.0);
    for (size_t i = k; i < n; ++i) v[i] = a[k * n + i];
    v[k] -= alpha;
    double vv = 0;
    for (size_t i = k; i < n; ++i) vv += v[i] * v[i];
    if (vv > 0) {
      for (size_t c = k; c < m; ++c) {
        double dot = 0;
        for (size_t i = k; i < n; ++i) dot += v[i] * a[c * n + i];
        const double f = 2.0 * dot / vv;
        for (size_t i = k; i < n; ++i) a[c * n + i] -= f * v[i];
      }
      double dot = 0;
      for (size_t i = k; i < n; ++i) dot += v[i] * b[i];
      const double f = 2.0 * dot / vv;
      for (size_t i = k; i < n; ++i) b[i] -= f * v[i];
    }
    rdiag[k] = a[k * n + k];
    ++rank;
  }
  if (rank < m) throw ConfigError("underdetermined: profile design matrix is rank deficient");
  // back substitution R x = Q^T b
  std::vector<double> x(m, 0.0);
  for (size_t k = m; k-- > 0;) {
    double s = b[k];
    for (size_t c = k + 1; c < m; ++c) s -= a[c * n + k] * x[c];
    x[k] = s / rdiag[k];
  }
  std::array<double, 3> full{0.0, 0.0, 0.0};
  for (size_t c = 0; c < m; ++c) full[static_cast<size_t>(active[perm[c]])] = x[c];
  return full;
}

}  // namespace

std::array<double, 3> fit_cost(const double* x1, const double* x2, const double* y, size_t n) {
  if (n < 3) throw ConfigError("underdetermined: need at least three profile samples");
  std::vector<double> design(3 * n), yy(y, y + n);
  for (size_t i = 0; i < n; ++i) {
    design[i] = 1.0;
    design[n + i] = x1[i];
    design[2 * n + i] = x2[i];
  }
  // Lengths spanning orders of magnitude: scale columns to unit norm.
  std::array<double, 3> scale{};
  for (int c = 0; c < 3; ++c) {
    double s = 0;
    for (size_t i = 0; i < n; ++i) s += design[c * n + i] * design[c * n + i];
    scale[c] = s > 0 ? std::sqrt(s) : 1.0;
    for (size_t i = 0; i < n; ++i) design[c * n + i] /= scale[c];
  }
  std::vector<int> active{0, 1, 2};
  std::array<double, 3> coef = solve_active(design, yy, n, active);
  while (true) {  // drop the most negative coefficient, refit
    int worst = -1;
    double worst_value = -1e-12;
    for (int c : active) {
      if (coef[c] < worst_value) {
        worst_value = coef[c];
        worst = c;
      }
    }
    if (worst < 0) break;
    active.erase(std::find(active.begin(), active.end(), worst));
    if (active.empty()) {
      coef = {0.0, 0.0, 0.0};
      break;
    }
    coef = solve_active(design, yy, n, active);
  }
  for (int c = 0; c < 3; ++c) coef[c] = std::max(coef[c], 0.0) / scale[c];
  return coef;
}

}  // namespace esp
