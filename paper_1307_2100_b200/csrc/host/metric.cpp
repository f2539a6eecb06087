// tc/metric.hpp: metric tensors and index raising / lowering on top of the
// contraction path (reference proj/src/metric.cpp:13-104: same checks, error
// texts and contraction layout; the Eigen FullPivLU it calls is restated
// below as a plain complete-pivoting elimination).
#include "tc/metric.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace tc {
namespace {

// Column-major n x n helper views.
struct Square {
  std::int64_t n;
  std::vector<double> a;
  explicit Square(std::int64_t n_) : n(n_), a(static_cast<std::size_t>(n_ * n_), 0.0) {}
  double& operator()(std::int64_t i, std::int64_t j) { return a[static_cast<std::size_t>(i + j * n)]; }
  double operator()(std::int64_t i, std::int64_t j) const {
    return a[static_cast<std::size_t>(i + j * n)];
  }
};

double one_norm(const Square& m) {  // largest absolute column sum
  double worst = 0.0;
  for (std::int64_t j = 0; j < m.n; ++j) {
    double s = 0.0;
    for (std::int64_t i = 0; i < m.n; ++i) s += std::fabs(m(i, j));
    worst = std::max(worst, s);
  }
  return worst;
}

// P A Q = L U with complete pivoting (the largest remaining entry becomes
// the pivot of every step), then A^-1 = Q U^-1 L^-1 P column by column.
// Returns false when the matrix is rank deficient: a pivot not above
// n * epsilon * |largest pivot| (FullPivLU's default threshold).
bool invert_full_pivot(const Square& src, Square& inv) {
  const std::int64_t n = src.n;
  Square lu = src;
  std::vector<std::int64_t> row_of(static_cast<std::size_t>(n)), col_of(static_cast<std::size_t>(n));
  std::iota(row_of.begin(), row_of.end(), 0);
  std::iota(col_of.begin(), col_of.end(), 0);
  double biggest_pivot = 0.0;
  std::int64_t nonzero = n;
  for (std::int64_t s = 0; s < n; ++s) {
    std::int64_t pr = s, pc = s;
    double best = -1.0;
    for (std::int64_t j = s; j < n; ++j)
      for (std::int64_t i = s; i < n; ++i)
        if (std::fabs(lu(i, j)) > best) {
          best = std::fabs(lu(i, j));
          pr = i;
          pc = j;
        }
    if (best == 0.0) {  // the remaining block is zero
      nonzero = s;
      break;
    }
    biggest_pivot = std::max(biggest_pivot, best);
    if (pr != s) {
      for (std::int64_t j = 0; j < n; ++j) std::swap(lu(s, j), lu(pr, j));
      std::swap(row_of[static_cast<std::size_t>(s)], row_of[static_cast<std::size_t>(pr)]);
    }
    if (pc != s) {
      for (std::int64_t i = 0; i < n; ++i) std::swap(lu(i, s), lu(i, pc));
      std::swap(col_of[static_cast<std::size_t>(s)], col_of[static_cast<std::size_t>(pc)]);
    }
    const double pivot = lu(s, s);
    for (std::int64_t i = s + 1; i < n; ++i) lu(i, s) /= pivot;
    for (std::int64_t j = s + 1; j < n; ++j) {
      const double u = lu(s, j);
      if (u == 0.0) continue;
      for (std::int64_t i = s + 1; i < n; ++i) lu(i, j) -= lu(i, s) * u;
    }
  }
  const double threshold =
      static_cast<double>(n) * std::numeric_limits<double>::epsilon() * biggest_pivot;
  std::int64_t rank = 0;
  for (std::int64_t s = 0; s < nonzero; ++s)
    if (std::fabs(lu(s, s)) > threshold) ++rank;
  if (rank != n) return false;

  std::vector<double> y(static_cast<std::size_t>(n));
  for (std::int64_t c = 0; c < n; ++c) {
    // solve A x = e_c: y = L^-1 P e_c, z = U^-1 y, x = Q z
    for (std::int64_t i = 0; i < n; ++i)
      y[static_cast<std::size_t>(i)] = row_of[static_cast<std::size_t>(i)] == c ? 1.0 : 0.0;
    for (std::int64_t j = 0; j < n; ++j) {
      const double yj = y[static_cast<std::size_t>(j)];
      if (yj == 0.0) continue;
      for (std::int64_t i = j + 1; i < n; ++i) y[static_cast<std::size_t>(i)] -= lu(i, j) * yj;
    }
    for (std::int64_t j = n - 1; j >= 0; --j) {
      y[static_cast<std::size_t>(j)] /= lu(j, j);
      const double zj = y[static_cast<std::size_t>(j)];
      for (std::int64_t i = 0; i < j; ++i) y[static_cast<std::size_t>(i)] -= lu(i, j) * zj;
    }
    for (std::int64_t j = 0; j < n; ++j)
      inv(col_of[static_cast<std::size_t>(j)], c) = y[static_cast<std::size_t>(j)];
  }
  return true;
}

MetricTensor empty_metric(std::int64_t n) {
  MetricTensor m;
  m.dimension = n;
  m.g = Tensor::zeros({n, n}, {Variance::Down, Variance::Down}, "g");
  m.g_inv = Tensor::zeros({n, n}, {Variance::Up, Variance::Up}, "ginv");
  return m;
}

// out[.., x', ..] = t[.., x, ..] * form[x, x'] with t's mode order kept: the
// contraction "t[i0..] = t[i0.., i<mode>, ..] * g[i<mode>, i<mode>p]"
// (reference src/metric.cpp:62-92), planned and executed like any other.
Tensor contract_mode(const Tensor& t, int mode, const Tensor& form, Variance expected,
                     const KernelBackend& backend) {
  if (mode < 0 || mode >= t.rank()) throw std::invalid_argument("mode out of range");
  if (t.variance(mode) != expected)
    throw std::invalid_argument(std::string("mode is already ") +
                                (expected == Variance::Up ? "lowered" : "raised"));
  if (t.extent(mode) != form.extent(0))
    throw std::invalid_argument("mode extent does not match metric dimension");

  const Variance turned = expected == Variance::Up ? Variance::Down : Variance::Up;
  ContractionSpec spec;
  spec.left.name = t.name().empty() ? "t" : t.name();
  spec.output.name = spec.left.name;
  spec.right.name = "g";
  std::string summed;
  for (int m = 0; m < t.rank(); ++m) {
    const std::string label = "i" + std::to_string(m);
    spec.left.indices.push_back({label, t.variance(m)});
    if (m != mode) {
      spec.output.indices.push_back({label, t.variance(m)});
    } else {
      summed = label;
      spec.output.indices.push_back({label + "p", turned});
    }
  }
  spec.right.indices.push_back({summed, form.variance(0)});
  spec.right.indices.push_back({summed + "p", form.variance(1)});

  const ValidatedContraction v = validate(spec, t, form);
  const ExecutionPlan p = plan(v);
  auto done = execute(p, v, t, form, backend);
  return std::move(done.first);
}

}  // namespace

MetricTensor invert_metric(const Tensor& g) {
  if (g.rank() != 2 || g.extent(0) != g.extent(1))
    throw std::invalid_argument("metric must be a square rank-2 tensor");
  const std::int64_t n = g.extent(0);
  Square G(n);
  std::copy(g.data(), g.data() + n * n, G.a.begin());

  double largest = 0.0, skew = 0.0;
  for (std::int64_t j = 0; j < n; ++j)
    for (std::int64_t i = 0; i < n; ++i) {
      largest = std::max(largest, std::fabs(G(i, j)));
      skew = std::max(skew, std::fabs(G(i, j) - G(j, i)));
    }
  if (skew > 1e-10 * std::max(1.0, largest)) throw std::invalid_argument("metric is not symmetric");

  Square inv(n);
  if (!invert_full_pivot(G, inv)) throw std::invalid_argument("metric is singular");
  const double cond = one_norm(G) * one_norm(inv);
  if (!(cond < 1e12)) throw std::invalid_argument("metric is numerically singular");

  MetricTensor m = empty_metric(n);
  std::copy(G.a.begin(), G.a.end(), m.g.data());
  std::copy(inv.a.begin(), inv.a.end(), m.g_inv.data());
  return m;
}

MetricTensor spherical_metric(double r, double theta) {
  const double s = std::sin(theta);
  if (!(r > 0.0) || s == 0.0)
    throw std::invalid_argument("spherical metric is singular at r=0 or sin(theta)=0");
  MetricTensor m = empty_metric(3);
  const double diag[3] = {1.0, r * r, r * r * s * s};
  for (std::int64_t i = 0; i < 3; ++i) {
    m.g.data()[i * 4] = diag[i];
    m.g_inv.data()[i * 4] = 1.0 / diag[i];
  }
  return m;
}

Tensor lower_index(const Tensor& t, int mode, const MetricTensor& m,
                   const KernelBackend& backend) {
  return contract_mode(t, mode, m.g, Variance::Up, backend);
}

Tensor raise_index(const Tensor& t, int mode, const MetricTensor& m,
                   const KernelBackend& backend) {
  return contract_mode(t, mode, m.g_inv, Variance::Down, backend);
}

}  // namespace tc
