// Metric tensors and index raising / lowering — a caller of the contraction
// path: reference proj/include/tc/metric.hpp:9-34 (same names, arguments and
// error behaviour). lower_index / raise_index build an ordinary two-tensor
// contraction and run it through validate -> plan -> execute, i.e. on the
// device with the b200 backend (or slice by slice with a caller's backend).
//
// invert_metric: the reference inverts with Eigen's FullPivLU, a third-party
// dependency that is not vendored in the reference tree (Eigen 3 >= 3.3,
// proj/CMakeLists.txt:13); csrc/host/metric.cpp restates that published
// algorithm (LU with complete pivoting, rank decided by |pivot| against
// n * epsilon * |largest pivot|). Parity of the inverse is unpinned at the bit
// level (no Eigen here to run); the tests pin it through g * g_inv = 1 and the
// reference tests' known answers.
#pragma once
#include "tc/contract.hpp"

namespace tc {

/// Symmetric nonsingular rank-2 tensor g (down, down) and its inverse
/// (up, up): g lowers an index, g_inv raises one.
struct MetricTensor {
  Tensor g;
  Tensor g_inv;
  std::int64_t dimension = 0;
};

/// Direct inversion. std::invalid_argument for a non-square or non-rank-2
/// input, asymmetry beyond 1e-10 (relative to max(1, max|g|)), a singular
/// matrix, or a 1-norm condition estimate of 1e12 or more.
MetricTensor invert_metric(const Tensor& g);

/// diag(1, r^2, r^2 sin^2(theta)) with its exact diagonal inverse;
/// std::invalid_argument at r <= 0 or sin(theta) == 0.
MetricTensor spherical_metric(double r, double theta);

/// Contracts mode `mode` (which must be Up) of t against g: that mode comes
/// out Down, every other mode and the mode order are unchanged.
Tensor lower_index(const Tensor& t, int mode, const MetricTensor& m,
                   const KernelBackend& backend);

/// The dual: mode `mode` (Down) against g_inv, coming out Up.
Tensor raise_index(const Tensor& t, int mode, const MetricTensor& m,
                   const KernelBackend& backend);

}  // namespace tc
