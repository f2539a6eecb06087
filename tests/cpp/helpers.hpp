// Operand binding like the reference's test helpers (tests/helpers.hpp:12-39):
// left seeded with `seed`, right with `seed + 1`.
#pragma once
#include <map>
#include <string>

#include "tc/contract.hpp"

namespace tst {

inline tc::Tensor operand(const tc::TensorExpr& te, const std::map<std::string, std::int64_t>& ext,
                          std::uint64_t seed) {
  std::vector<std::int64_t> e;
  std::vector<tc::Variance> v;
  for (const auto& ix : te.indices) {
    e.push_back(ext.at(ix.label));
    v.push_back(ix.var);
  }
  return tc::Tensor::seeded_random(e, v, seed, te.name);
}

struct Bound {
  tc::ContractionSpec spec;
  tc::Tensor left, right;
  tc::ValidatedContraction v;
};

inline Bound bind_expr(const std::string& expr, const std::map<std::string, std::int64_t>& ext,
                       std::uint64_t seed = 1, bool positional = false) {
  Bound b{tc::parse(expr, positional), {}, {}, {}};
  b.left = operand(b.spec.left, ext, seed);
  b.right = operand(b.spec.right, ext, seed + 1);
  b.v = tc::validate(b.spec, b.left, b.right);
  return b;
}

}  // namespace tst
