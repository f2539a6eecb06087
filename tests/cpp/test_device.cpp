// Executor and backend suites restated from the reference's doctest files
// (tests/test_executor.cpp, tests/test_kernels.cpp) against the engine's
// device path: tc::execute with make_backend("b200"). Requires a B200.
#include <cstring>
#include <random>

#include "harness.hpp"
#include "helpers.hpp"
#include "tc/executor.hpp"
#include "tc/kernels.hpp"
#include "tc/metric.hpp"
#include "tc/oracle.hpp"

using namespace tc;
using tst::bind_expr;

namespace {
const auto kBackend = make_backend("b200");

// direct nested summation (src/oracle.cpp:32-94 order) for small cases
Tensor naive(const ValidatedContraction& v, const Tensor& L, const Tensor& R) {
  Tensor out(v.output_extents(), v.output_variance());
  std::vector<int> fr;
  for (const auto& ix : v.spec.output.indices) fr.push_back(v.label_index(ix.label));
  std::vector<std::int64_t> fc(fr.size(), 0);
  auto lstr = [&](int li) {
    const auto& i = v.labels[li];
    return i.left_mode >= 0 ? stride_of(L, i.left_mode) : 0;
  };
  auto rstr = [&](int li) {
    const auto& i = v.labels[li];
    return i.right_mode >= 0 ? stride_of(R, i.right_mode) : 0;
  };
  for (std::int64_t o = 0; o < out.size(); ++o) {
    std::int64_t t = o, lb = 0, rb = 0;
    for (std::size_t i = 0; i < fr.size(); ++i) {
      const std::int64_t e = v.labels[fr[i]].extent, c = t % e;
      t /= e;
      lb += c * lstr(fr[i]);
      rb += c * rstr(fr[i]);
    }
    std::int64_t total = 1;
    for (int ci : v.contracted) total *= v.labels[ci].extent;
    double acc = 0;
    for (std::int64_t q = 0; q < total; ++q) {
      std::int64_t u = q, lo = lb, ro = rb;
      for (int ci : v.contracted) {
        const std::int64_t e = v.labels[ci].extent, c = u % e;
        u /= e;
        lo += c * lstr(ci);
        ro += c * rstr(ci);
      }
      acc += L.data()[lo] * R.data()[ro];
    }
    out.data()[o] = acc;
  }
  return out;
}
}  // namespace

TEST_CASE("plain matrix product runs as a single device launch") {  // test_executor.cpp:20-30
  const auto b = bind_expr("C[+i,-j] = A[+i,+h] * B[-h,-j]", {{"i", 2}, {"j", 2}, {"h", 2}});
  const auto p = plan(b.v);
  auto [result, stats] = execute(p, b.v, b.left, b.right, *kBackend);
  CHECK(stats.kernel_calls == 1);
  CHECK(stats.packed_bytes == 0);
  CHECK(stats.flops == p.flops);
  CHECK(max_rel_error(result, naive(b.v, b.left, b.right)) <= 1e-15);
}

TEST_CASE("crossed stride-1 contraction permutes and matches the oracle") {
  const auto b = bind_expr("R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]",
                           {{"a", 4}, {"b", 4}, {"g", 4}, {"e", 4}});
  const auto p = plan(b.v);
  REQUIRE(p.kernel == KernelKind::CopyGemm);
  auto [result, stats] = execute(p, b.v, b.left, b.right, *kBackend);
  CHECK(stats.packed_bytes > 0);
  CHECK(max_rel_error(result, naive(b.v, b.left, b.right)) <= 1e-12);
}

TEST_CASE("full contraction to a scalar") {  // test_executor.cpp:43-54
  const auto b = bind_expr("K[] = T[+a,+b,+g] * S[-a,-b,-g]", {{"a", 3}, {"b", 3}, {"g", 3}});
  auto [result, stats] = execute(plan(b.v), b.v, b.left, b.right, *kBackend);
  double expect = 0;
  for (std::int64_t i = 0; i < b.left.size(); ++i) expect += b.left.data()[i] * b.right.data()[i];
  CHECK(std::abs(result.at({}) - expect) <= 1e-13 * std::abs(expect) + 1e-15);
}

TEST_CASE("auto plans match the oracle across a randomized family") {
  std::mt19937_64 rng(31337);
  const char* exprs[] = {"R[+a,-e] = A[+a,+b,+g] * B[-e,-b,-g]",
                         "R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]",
                         "R[+a,+b,+c,+d] = X[+i,+a,+j,+b] * Y[-j,+c,-i,+d]",
                         "R[+g] = T[+a,+b,+g] * G[-a,-b]"};
  for (int it = 0; it < 40; ++it) {
    std::map<std::string, std::int64_t> ext;
    for (const char* l : {"a", "b", "c", "d", "e", "g", "i", "j"})
      ext[l] = 1 + static_cast<std::int64_t>(rng() % 6);
    const auto b = bind_expr(exprs[it % 4], ext, it);
    auto [r, s] = execute(plan(b.v), b.v, b.left, b.right, *kBackend);
    CHECK(max_rel_error(r, naive(b.v, b.left, b.right)) <= 1e-12);
  }
}

TEST_CASE("every enumerated slicing computes the same tensor") {  // test_executor.cpp:89-102
  const auto b = bind_expr("C[+i,-j] = A[+i,+h] * B[-h,-j]", {{"i", 3}, {"j", 3}, {"h", 3}});
  const auto runs = execute_all_slicings(b.v, b.left, b.right, *kBackend);
  REQUIRE(!runs.empty());
  for (const auto& r : runs) CHECK(max_rel_error(r.result, runs[0].result) <= 1e-12);
  CHECK_THROWS_AS(execute_all_slicings(b.v, b.left, b.right, *kBackend, 10), resource_limit_error);
}

TEST_CASE("worker count does not change the result") {  // test_executor.cpp:209-219
  const auto b = bind_expr("R[+a,+b,+c,+d] = X[+i,+a,+j,+b] * Y[-i,+c,-j,+d]",
                           {{"a", 3}, {"b", 4}, {"c", 3}, {"d", 4}, {"i", 3}, {"j", 3}});
  const auto p = plan(b.v);
  auto [r1, s1] = execute(p, b.v, b.left, b.right, *kBackend, 1);
  auto [r2, s2] = execute(p, b.v, b.left, b.right, *kBackend, 3);
  CHECK(tensor_hash(r1) == tensor_hash(r2));
}

TEST_CASE("extent drift between planning and execution is rejected") {  // :221-229
  const auto b = bind_expr("C[+i,-j] = A[+i,+h] * B[-h,-j]", {{"i", 3}, {"j", 3}, {"h", 3}});
  const auto p = plan(b.v);
  const auto b2 = bind_expr("C[+i,-j] = A[+i,+h] * B[-h,-j]", {{"i", 4}, {"j", 4}, {"h", 4}});
  CHECK_THROWS_AS(execute(p, b2.v, b2.left, b2.right, *kBackend), std::invalid_argument);
}

TEST_CASE("device faults surface with the contraction attached") {  // :240-291
  const auto b = bind_expr("R[+a,-e] = A[+a,+b,+g] * B[-e,-b,-g]",
                           {{"a", 3}, {"b", 3}, {"g", 3}, {"e", 3}});
  B200Options o;
  o.fail_after_launches = 0;
  const auto failing = make_b200_backend(o);
  try {
    execute(plan(b.v), b.v, b.left, b.right, *failing);
    CHECK(false);
  } catch (const std::runtime_error& e) {
    const std::string what = e.what();
    CHECK(what.find("synthetic device fault") != std::string::npos);
    CHECK(what.find("R[+a,-e]") != std::string::npos);
  }
}

TEST_CASE("tc/oracle.hpp: contract_naive equals the direct sum, refuses above its cap") {
  const auto b = bind_expr("R[+a,+b,+c,+d] = X[+i,+a,+j,+b] * Y[-j,+c,-i,+d]",
                           {{"a", 2}, {"b", 3}, {"c", 2}, {"d", 3}, {"i", 2}, {"j", 3}});
  OracleStats st;
  const Tensor got = contract_naive(b.v, b.left, b.right, 1000000000, &st);
  const Tensor want = naive(b.v, b.left, b.right);
  CHECK(std::memcmp(got.data(), want.data(), static_cast<std::size_t>(got.size()) * 8) == 0);
  CHECK(st.multiply_adds == 2 * 3 * 2 * 3 * 2 * 3);
  CHECK_THROWS_AS(contract_naive(b.v, b.left, b.right, 10), resource_limit_error);
}

TEST_CASE("backend gemm/gemv/ger/dot known answers on host pointers") {  // test_kernels.cpp
  const std::vector<double> A{1, 3, 2, 4}, B{5, 7, 6, 8};
  std::vector<double> C(4, 0);
  kBackend->gemm(false, false, 2, 2, 2, 1.0, A.data(), 2, B.data(), 2, 0.0, C.data(), 2);
  CHECK((C == std::vector<double>{19, 43, 22, 50}));
  std::vector<double> C1{1, 1, 1, 1};
  kBackend->gemm(false, false, 2, 2, 2, 1.0, A.data(), 2, B.data(), 2, 1.0, C1.data(), 2);
  CHECK((C1 == std::vector<double>{20, 44, 23, 51}));
  std::vector<double> x2{1, 1}, y2(2, 0);
  kBackend->gemv(false, 2, 2, 1.0, A.data(), 2, x2.data(), 1, 0.0, y2.data(), 1);
  CHECK((y2 == std::vector<double>{3, 7}));
  std::vector<double> G(4, 0);
  const std::vector<double> gx{1, 2}, gy{3, 4};
  kBackend->ger(2, 2, 1.0, gx.data(), 1, gy.data(), 1, G.data(), 2);
  CHECK((G == std::vector<double>{3, 6, 4, 8}));
  const std::vector<double> dx{1, 2, 3}, dy{4, 5, 6};
  CHECK(kBackend->dot(3, dx.data(), 1, dy.data(), 1) == 32.0);
  std::vector<double> Z(4);
  CHECK_THROWS_AS(kBackend->gemm(false, false, 2, 2, 2, 1.0, Z.data(), 1, Z.data(), 2, 0.0,
                                 Z.data(), 2),
                  std::invalid_argument);
}

// ------------------------------------------------------ metric (tc/metric.hpp)
// lower_index / raise_index on the device (reference tests/test_metric.cpp)
namespace {
MetricTensor dense3() {
  return invert_metric(Tensor::from_values({3, 3}, {Variance::Down, Variance::Down},
                                           {4, 1, 0.5, 1, 3, 0.25, 0.5, 0.25, 2}));
}
}  // namespace

TEST_CASE("metric lowering on the device: diagonal products, round trip, commuting modes") {
  const double r = 2.0, th = M_PI / 2;
  const auto sph = spherical_metric(r, th);
  const Tensor S = Tensor::seeded_random({3, 3}, {Variance::Up, Variance::Up}, 17, "S");
  const Tensor low = lower_index(lower_index(S, 0, sph, *kBackend), 1, sph, *kBackend);
  const double d[3] = {1.0, r * r, r * r * std::sin(th) * std::sin(th)};
  for (std::int64_t i = 0; i < 3; ++i)
    for (std::int64_t j = 0; j < 3; ++j)
      CHECK(std::fabs(low.at({i, j}) - d[i] * d[j] * S.at({i, j})) <= 1e-12 * 16);
  CHECK(low.variance(0) == Variance::Down);
  CHECK(low.variance(1) == Variance::Down);

  const auto m = dense3();
  const Tensor t =
      Tensor::seeded_random({3, 4, 3}, {Variance::Up, Variance::Down, Variance::Up}, 5);
  for (const int mode : {0, 2}) {
    const Tensor back = raise_index(lower_index(t, mode, m, *kBackend), mode, m, *kBackend);
    CHECK(max_rel_error(back, t) <= 1e-10);
  }
  // a metric dimension that spans several tiles: 200 x 200 SPD, rank-3 tensor
  const std::int64_t n = 200;
  Tensor g = Tensor::zeros({n, n}, {Variance::Down, Variance::Down});
  const Tensor noise = Tensor::seeded_random({n, n}, {Variance::Down, Variance::Down}, 77);
  for (std::int64_t i = 0; i < n; ++i)
    for (std::int64_t j = 0; j < n; ++j)
      g.data()[i + j * n] = (i == j ? 8.0 : 0.0) +
                            0.01 * (noise.data()[i + j * n] + noise.data()[j + i * n]);
  const auto big = invert_metric(g);
  const Tensor w = Tensor::seeded_random({37, n, 5}, {Variance::Down, Variance::Up, Variance::Up}, 6);
  const Tensor wl = lower_index(w, 1, big, *kBackend);
  CHECK(wl.variance(1) == Variance::Down);
  // against the direct sum over the contracted mode
  double worst = 0, scale = 1;
  for (std::int64_t c = 0; c < 5; ++c)
    for (std::int64_t x = 0; x < n; x += 17)
      for (std::int64_t a = 0; a < 37; a += 5) {
        double acc = 0;
        for (std::int64_t y = 0; y < n; ++y) acc += w.at({a, y, c}) * big.g.at({y, x});
        worst = std::max(worst, std::fabs(acc - wl.at({a, x, c})));
        scale = std::max(scale, std::fabs(acc));
      }
  CHECK(worst / scale <= 1e-12);
  CHECK(max_rel_error(raise_index(wl, 1, big, *kBackend), w) <= 1e-10);
}

TEST_CASE("metric placements: both routes agree and all six match the oracle") {  // :153-218
  const auto m = dense3();
  const Tensor T = Tensor::seeded_random({2, 2, 3}, std::vector<Variance>(3, Variance::Up), 21, "T");
  const Tensor S = Tensor::seeded_random({3, 2}, std::vector<Variance>(2, Variance::Up), 22, "S");
  const Tensor Tl = lower_index(T, 2, m, *kBackend);
  const auto v1 = validate(parse("R[+a,+b,+r] = T[+a,+b,-s] * S[+s,+r]"), Tl, S);
  const Tensor r1 = execute(plan(v1), v1, Tl, S, *kBackend).first;
  const Tensor Sl = lower_index(S, 0, m, *kBackend);
  const auto v2 = validate(parse("R[+a,+b,+r] = T[+a,+b,+s] * S[-s,+r]"), T, Sl);
  const Tensor r2 = execute(plan(v2), v2, T, Sl, *kBackend).first;
  CHECK(max_rel_error(r1, r2) <= 1e-12);

  const Tensor T3 = Tensor::seeded_random({3, 3, 3}, std::vector<Variance>(3, Variance::Up), 33, "T");
  const Tensor S3 = Tensor::seeded_random({3, 3}, std::vector<Variance>(2, Variance::Up), 34, "S");
  const char* names[3] = {"a", "b", "c"};
  for (int t_mode = 0; t_mode < 3; ++t_mode)
    for (int s_mode = 0; s_mode < 2; ++s_mode) {
      const Tensor low = lower_index(T3, t_mode, m, *kBackend);
      ContractionSpec spec;
      spec.left.name = "T";
      spec.right.name = "S";
      spec.output.name = "R";
      for (int k = 0; k < 3; ++k) {
        if (k == t_mode) {
          spec.left.indices.push_back({"s", Variance::Down});
        } else {
          spec.left.indices.push_back({names[k], Variance::Up});
          spec.output.indices.push_back({names[k], Variance::Up});
        }
      }
      for (int k = 0; k < 2; ++k) {
        if (k == s_mode) {
          spec.right.indices.push_back({"s", Variance::Up});
        } else {
          spec.right.indices.push_back({"r", Variance::Up});
          spec.output.indices.push_back({"r", Variance::Up});
        }
      }
      const auto v = validate(spec, low, S3);
      const Tensor got = execute(plan(v), v, low, S3, *kBackend).first;
      CHECK(max_rel_error(got, contract_naive(v, low, S3)) <= 1e-12);
      CHECK(max_rel_error(got, naive(v, low, S3)) <= 1e-12);
    }
}

TH_MAIN
