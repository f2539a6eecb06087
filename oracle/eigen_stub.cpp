// TEST INFRASTRUCTURE ONLY. Eigen 3 is absent from this image, so the
// reference's Eigen adapter (src/kernels_eigen.cpp) cannot be compiled. The
// reference factory make_backend (src/kernels_reference.cpp:158-162) still
// names make_eigen_backend, so this stub satisfies the link and fails loudly.
#include <stdexcept>

#include "tc/kernels.hpp"

namespace tc {
std::unique_ptr<KernelBackend> make_eigen_backend() {
  throw std::invalid_argument("external (Eigen) backend not available in this build");
}
}  // namespace tc
