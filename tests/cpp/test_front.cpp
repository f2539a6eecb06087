// Host-front suites restated from the reference's doctest files
// (tests/test_tensor.cpp, test_expr.cpp, test_planner.cpp) against the
// engine's tc:: API. CPU only.
#include <cstring>
#include <set>

#include "harness.hpp"
#include "helpers.hpp"
#include "tc/metric.hpp"
#include "tc/tensor_io.hpp"

using namespace tc;
using tst::bind_expr;

namespace {
const std::map<std::string, std::int64_t> kSq{{"a", 4}, {"b", 4}, {"g", 4}, {"e", 4}};
const std::map<std::string, std::int64_t> kSq3{{"a", 3}, {"b", 3}, {"g", 3}};

bool has_option(const std::vector<SlicingOption>& opts, const SlicingVector& sl,
                const SlicingVector& sr, KernelKind k) {
  for (const auto& o : opts)
    if (o.s_left == sl && o.s_right == sr && o.report.kernel == k) return true;
  return false;
}
Tensor mk(std::vector<std::int64_t> ext, const std::string& vars) {
  std::vector<Variance> v;
  for (char c : vars) v.push_back(c == '+' ? Variance::Up : Variance::Down);
  return Tensor::zeros(ext, v);
}
}  // namespace

// ------------------------------------------------------------ tensor (L0)
TEST_CASE("column-major layout and strides") {  // test_tensor.cpp:19-66
  Tensor t = Tensor::sequential({2, 3, 4}, {Variance::Up, Variance::Down, Variance::Up});
  CHECK(t.at({1, 0, 0}) == 1.0);
  CHECK(t.at({0, 1, 0}) == 2.0);
  CHECK(t.at({0, 0, 1}) == 6.0);
  CHECK(stride_of(t, 0) == 1);
  CHECK(stride_of(t, 1) == 2);
  CHECK(stride_of(t, 2) == 6);
  CHECK_THROWS_AS(t.at({2, 0, 0}), std::out_of_range);
  CHECK_THROWS_AS(Tensor({0}, {Variance::Up}), std::invalid_argument);
}

TEST_CASE("seeded determinism") {  // test_tensor.cpp:33-45
  auto a = Tensor::seeded_random({5, 7}, {Variance::Up, Variance::Up}, 9);
  auto b = Tensor::seeded_random({5, 7}, {Variance::Up, Variance::Up}, 9);
  auto c = Tensor::seeded_random({5, 7}, {Variance::Up, Variance::Up}, 10);
  CHECK(tensor_hash(a) == tensor_hash(b));
  CHECK(tensor_hash(a) != tensor_hash(c));
  for (std::int64_t i = 0; i < a.size(); ++i) CHECK(a.data()[i] >= -1.0 && a.data()[i] <= 1.0);
}

TEST_CASE("slice views alias and pack") {  // test_tensor.cpp:83-224
  Tensor t = Tensor::sequential({3, 4, 5}, {Variance::Up, Variance::Up, Variance::Up});
  auto v = slice_view(t, {0, 1, 0}, {2});
  CHECK(v.rank() == 2);
  CHECK(v.at({1, 3}) == t.at({1, 2, 3}));
  auto pm = pack_slice(v);
  CHECK_FALSE(pm.copied);
  CHECK(pm.leading_dimension == 12);
  auto w = slice_view(t, {1, 0, 0}, {1});
  auto pw = pack_slice(w);
  CHECK(pw.copied);
  CHECK(pw.data[2 + 3 * 4] == t.at({1, 2, 3}));
}

// ------------------------------------------------------------ expr (L1)
TEST_CASE("parse identifies contracted and free labels") {  // test_expr.cpp:20-31
  const auto s = parse("R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]");
  CHECK(s.left.name == "A");
  CHECK(s.output.indices.size() == 2);
  CHECK(s.left.indices[1].label == "b");
  CHECK(s.right.indices[0].var == Variance::Down);
  CHECK_THROWS_AS(parse("R[+a,-e] = A[+a,+b,+g] * B[-g,-a,-e]"), parse_error);
}

TEST_CASE("validate binds extents and deltas") {  // test_expr.cpp:125-200
  const auto s = parse("R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]");
  const auto v = validate(s, mk({4, 5, 6}, "+++"), mk({6, 4, 7}, "---"));
  CHECK(v.delta_left == 1);
  CHECK(v.delta_right == 1);
  CHECK(v.p == 2);
  CHECK(v.labels[v.label_index("e")].extent == 7);
  CHECK_THROWS_AS(validate(s, mk({4, 5, 6}, "+++"), mk({6, 9, 7}, "---")), std::invalid_argument);
  const auto sp = parse("R[+a] = T[+a,+b] * x[-b]", true);
  validate(sp, mk({3, 4}, "+-"), mk({4}, "-"));
  CHECK_THROWS_AS(validate(parse("R[+a] = T[+a,+b] * x[-b]"), mk({3, 4}, "+-"), mk({4}, "-")),
                  std::invalid_argument);
}

TEST_CASE("parse of unparse is the identity") {  // test_expr.cpp:79-123
  for (const char* e : {"R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]", "K[] = T[+a,+b,+g] * S[-a,-b,-g]",
                        "C[+i,-j] = A[+i,+h] * B[-h,-j]"}) {
    const auto s = parse(e);
    CHECK(parse(unparse(s)) == s);
    CHECK(unparse(s) == e);
  }
}

TEST_CASE("flop count") {  // test_expr.cpp:202-217
  CHECK(flop_count(validate(parse("R[+a,-e] = A[+a,+b,+g] * B[-e,-b,-g]"), mk({10, 10, 10}, "+++"),
                            mk({10, 10, 10}, "---"))) == 20000);
  CHECK(flop_count(validate(parse("K[] = T[+a,+b,+g] * S[-a,-b,-g]"), mk({3, 3, 3}, "+++"),
                            mk({3, 3, 3}, "---"))) == 54);
}

// ------------------------------------------------------------ planner (L2)
TEST_CASE("classify the taxonomy anchor cases") {  // test_planner.cpp:27-45
  CHECK(classify(bind_expr("K[] = T[+a,+b,+g] * S[-a,-b,-g]", kSq3).v) == ContractionClass::C1);
  CHECK(classify(bind_expr("R[+a] = T[+a,+b,+g] * G[-b,-g]", kSq3).v) == ContractionClass::C2);
  CHECK(classify(bind_expr("R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]", kSq).v) == ContractionClass::C31);
  CHECK(classify(bind_expr("R[+a,-e] = A[+a,+b,+g] * B[-e,-b,-g]", kSq).v) == ContractionClass::C32);
}

TEST_CASE("check_requirements catalog") {  // test_planner.cpp:79-129
  const auto b = bind_expr("R[+a,-e] = A[+a,+b,+g] * B[-e,-b,-g]", kSq);
  const auto rep = check_requirements(b.v, {0, 1, 0}, {0, 1, 0});
  CHECK(rep.r1_ok && rep.r2_ok && rep.r3_ok);
  CHECK(rep.kernel == KernelKind::Gemm);
  const auto c = bind_expr("R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]", kSq);
  CHECK(check_requirements(c.v, {0, 0, 1}, {1, 0, 1}).kernel == KernelKind::Gemv);
  CHECK(check_requirements(c.v, {1, 0, 1}, {1, 1, 0}).kernel == KernelKind::Ger);
  CHECK_THROWS_AS(check_requirements(b.v, {0, 1, 0}, {0, 0, 0}), std::invalid_argument);
}

TEST_CASE("matmul enumeration: four decompositions plus GEMM") {  // test_planner.cpp:137-148
  const auto b = bind_expr("C[+i,-j] = A[+i,+h] * B[-h,-j]", {{"i", 3}, {"j", 4}, {"h", 5}});
  const auto opts = enumerate_slicings(b.v);
  CHECK(has_option(opts, {0, 0}, {0, 0}, KernelKind::Gemm));
  CHECK(has_option(opts, {1, 0}, {0, 0}, KernelKind::Gemv));
  CHECK(has_option(opts, {0, 0}, {0, 1}, KernelKind::Gemv));
  CHECK(has_option(opts, {0, 1}, {1, 0}, KernelKind::Ger));
  CHECK(has_option(opts, {1, 0}, {0, 1}, KernelKind::Dot));
  for (std::size_t i = 1; i < opts.size(); ++i)
    CHECK(std::tie(opts[i - 1].s_left, opts[i - 1].s_right) <
          std::tie(opts[i].s_left, opts[i].s_right));
}

TEST_CASE("class 3.2 auto plan accumulates over the sliced contracted label") {
  // test_planner.cpp:226-239
  const auto b = bind_expr("R[+a,-e] = A[+a,+b,+g] * B[-e,-b,-g]",
                           {{"a", 5}, {"b", 4}, {"g", 3}, {"e", 6}});
  const auto p = plan(b.v);
  CHECK(p.kernel == KernelKind::Gemm);
  REQUIRE(p.loop_nest.size() == 1);
  CHECK(p.loop_nest[0].contracted);
  CHECK(b.v.labels[p.loop_nest[0].label].label == "g");
  CHECK(p.copies.empty());
  CHECK(p.flops == flop_count(b.v));
}

TEST_CASE("recipes and forced-GEMM errors") {  // test_planner.cpp:244-307
  CHECK(plan(bind_expr("K[] = T[+a,+b,+g] * S[-a,-b,-g]", kSq3).v).kernel == KernelKind::Dot);
  CHECK(plan(bind_expr("R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]", kSq).v).kernel ==
        KernelKind::CopyGemm);
  CHECK_THROWS_WITH_AS(plan(bind_expr("K[] = T[+a,+b,+g] * S[-a,-b,-g]", kSq3).v,
                            PlanPolicy::force_kernel(KernelKind::Gemm)),
                       "kernel unreachable: R3 violated", kernel_unreachable_error);
  CHECK_THROWS_WITH_AS(plan(bind_expr("R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]", kSq).v,
                            PlanPolicy::force_kernel(KernelKind::Gemm)),
                       "kernel unreachable: R1 violated", kernel_unreachable_error);
  CHECK_THROWS_WITH_AS(plan(bind_expr("R[+a] = T[+a,+b] * x[-b]", {{"a", 4}, {"b", 5}}).v,
                            PlanPolicy::force_kernel(KernelKind::Gemm)),
                       "kernel unreachable: R2 violated", kernel_unreachable_error);
}

TEST_CASE("plan report renders deterministically") {  // test_planner.cpp:334-349
  const auto b = bind_expr("R[+a,-e] = A[+a,+b,+g] * B[-e,-b,-g]", kSq);
  CHECK(render_plan(plan(b.v), b.v) ==
        "class: 3.2\ndelta: (1, 1)\ns_left: (0, 0, 1)\ns_right: (0, 0, 1)\ns_output: (0, 0)\n"
        "kernel: GEMM\nloop_nest: g:contracted\nkernel_map: M=a N=e K=b transA=0 transB=1\n"
        "copies: 0\nflops: 512\n");
}

TEST_CASE("relayout advice turns a crossed contraction into a direct one") {
  const auto b = bind_expr("R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]", kSq);
  const auto adv = relayout_advice(b.v);
  REQUIRE(adv.has_value());
  CHECK(adv->find("class 3.2") != std::string::npos);
  CHECK_FALSE(relayout_advice(bind_expr("R[+a,-e] = A[+a,+b,+g] * B[-e,-b,-g]", kSq).v));
}

TEST_CASE("loop nest and kernel map partition the labels (BASELINE configs)") {
  const std::pair<const char*, std::map<std::string, std::int64_t>> cfgs[] = {
      {"C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", {{"i", 8}, {"j", 8}, {"k", 4}, {"l", 4}}},
      {"C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", {{"a", 4}, {"b", 4}, {"c", 4}, {"k", 4}}},
      {"C[+a,+b,+c,+d] = A[+a,+k,+c,+l] * B[-l,+b,-k,+d]",
       {{"a", 4}, {"b", 4}, {"c", 4}, {"d", 4}, {"k", 2}, {"l", 2}}}};
  for (const auto& [e, ext] : cfgs) {
    const auto b = bind_expr(e, ext);
    CHECK(classify(b.v) == ContractionClass::C32);  // all BASELINE configs 3.2
    const auto p = plan(b.v);
    std::set<int> seen;
    for (const auto& l : p.loop_nest) CHECK(seen.insert(l.label).second);
    for (int k : {p.kernel_map.m_label, p.kernel_map.n_label, p.kernel_map.k_label})
      if (k >= 0) CHECK(seen.insert(k).second);
    CHECK(seen.size() == b.v.labels.size());
  }
}

TEST_CASE("only the device backend exists") {
  CHECK(make_backend("b200")->name() == "b200");
  CHECK_THROWS_AS(make_backend("reference"), std::invalid_argument);
  CHECK_THROWS_AS(make_backend("nope"), std::invalid_argument);
  // the reference's factories link, and name the replacement
  CHECK_THROWS_AS(make_reference_backend(), std::invalid_argument);
  CHECK_THROWS_AS(make_eigen_backend(), std::invalid_argument);
}

// ------------------------------------------- caller-supplied KernelBackend
// execute() drives any non-B200 backend slice by slice, as the reference does
// (src/executor.cpp:102-369). A plain host BLAS written here (test code).
namespace {
class HostBlas : public KernelBackend {
 public:
  mutable std::int64_t calls = 0;
  const std::string& name() const override {
    static const std::string n = "host-test";
    return n;
  }
  bool supports_transpose() const override { return true; }
  void gemm(bool ta, bool tb, std::int64_t m, std::int64_t n, std::int64_t k, double alpha,
            const double* a, std::int64_t lda, const double* b, std::int64_t ldb, double beta,
            double* c, std::int64_t ldc) const override {
    ++calls;
    for (std::int64_t j = 0; j < n; ++j)
      for (std::int64_t i = 0; i < m; ++i) {
        double s = 0;
        for (std::int64_t p = 0; p < k; ++p)
          s += (ta ? a[p + i * lda] : a[i + p * lda]) * (tb ? b[j + p * ldb] : b[p + j * ldb]);
        c[i + j * ldc] = alpha * s + (beta == 0 ? 0.0 : beta * c[i + j * ldc]);
      }
  }
  void gemv(bool trans, std::int64_t m, std::int64_t n, double alpha, const double* a,
            std::int64_t lda, const double* x, std::int64_t incx, double beta, double* y,
            std::int64_t incy) const override {
    ++calls;
    const std::int64_t rows = trans ? n : m, inner = trans ? m : n;
    for (std::int64_t r = 0; r < rows; ++r) {
      double s = 0;
      for (std::int64_t q = 0; q < inner; ++q)
        s += (trans ? a[q + r * lda] : a[r + q * lda]) * x[q * incx];
      y[r * incy] = alpha * s + (beta == 0 ? 0.0 : beta * y[r * incy]);
    }
  }
  void ger(std::int64_t m, std::int64_t n, double alpha, const double* x, std::int64_t incx,
           const double* y, std::int64_t incy, double* a, std::int64_t lda) const override {
    ++calls;
    for (std::int64_t j = 0; j < n; ++j)
      for (std::int64_t i = 0; i < m; ++i) a[i + j * lda] += alpha * x[i * incx] * y[j * incy];
  }
  double dot(std::int64_t k, const double* x, std::int64_t incx, const double* y,
             std::int64_t incy) const override {
    ++calls;
    double s = 0;
    for (std::int64_t i = 0; i < k; ++i) s += x[i * incx] * y[i * incy];
    return s;
  }
};

class FailingBlas : public HostBlas {
 public:
  explicit FailingBlas(int after) : after_(after) {}
  void gemm(bool ta, bool tb, std::int64_t m, std::int64_t n, std::int64_t k, double alpha,
            const double* a, std::int64_t lda, const double* b, std::int64_t ldb, double beta,
            double* c, std::int64_t ldc) const override {
    if (calls >= after_) throw std::runtime_error("injected backend failure");
    HostBlas::gemm(ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc);
  }

 private:
  int after_;
};

// brute force over every label (test code)
std::vector<double> brute(const tst::Bound& b) {
  const auto& v = b.v;
  std::vector<double> out(static_cast<std::size_t>(
      [&] { std::int64_t n = 1; for (auto e : v.output_extents()) n *= e; return n; }()), 0.0);
  const std::size_t nl = v.labels.size();
  std::vector<std::int64_t> at(nl, 0);
  for (;;) {
    std::int64_t lo = 0, ro = 0, oo = 0;
    for (std::size_t i = 0; i < nl; ++i) {
      const auto& li = v.labels[i];
      if (li.left_mode >= 0) lo += at[i] * stride_of(b.left, li.left_mode);
      if (li.right_mode >= 0) ro += at[i] * stride_of(b.right, li.right_mode);
      if (li.output_mode >= 0) {
        std::int64_t s = 1;
        for (int m = 0; m < li.output_mode; ++m) s *= v.output_extents()[static_cast<std::size_t>(m)];
        oo += at[i] * s;
      }
    }
    out[static_cast<std::size_t>(oo)] += b.left.data()[lo] * b.right.data()[ro];
    std::size_t k = 0;
    for (; k < nl; ++k) {
      if (++at[k] < v.labels[k].extent) break;
      at[k] = 0;
    }
    if (k == nl) break;
  }
  return out;
}

double max_rel(const Tensor& got, const std::vector<double>& want) {
  double scale = 1, worst = 0;
  for (double w : want) scale = std::max(scale, std::fabs(w));
  for (std::size_t i = 0; i < want.size(); ++i)
    worst = std::max(worst, std::fabs(got.data()[i] - want[i]));
  return worst / scale;
}
}  // namespace

TEST_CASE("a caller's backend runs every slicing slice by slice") {  // test_executor.cpp:89-102
  const char* exprs[] = {
      "C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]",
      "C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]",
      "C[+a,+b,+c,+d] = A[+a,+k,+c,+l] * B[-l,+b,-k,+d]",
      "R[+a,-e] = A[+a,+b,+g] * B[-e,-b,-g]",
      "R[+a] = T[+a,+b,+g] * G[-b,-g]",
      "K[] = T[+a,+b,+g] * S[-a,-b,-g]",
      "C[+b,+a] = A[+k,+a] * B[-k,+b]",
  };
  const std::map<std::string, std::int64_t> ext{{"i", 5}, {"j", 4}, {"k", 3}, {"l", 2},
                                               {"a", 4}, {"b", 3}, {"c", 2}, {"d", 3},
                                               {"e", 2}, {"g", 3}};
  HostBlas be;
  for (const char* e : exprs) {
    const auto b = bind_expr(e, ext);
    const auto want = brute(b);
    for (const auto& o : enumerate_slicings(b.v)) {
      ExecutionPlan p;
      try {
        p = plan(b.v, PlanPolicy::force_slicing(o.s_left, o.s_right));
      } catch (const kernel_unreachable_error&) {
        continue;
      }
      be.calls = 0;
      const auto [res, st] = execute(p, b.v, b.left, b.right, be);
      CHECK(max_rel(res, want) <= 1e-13);
      CHECK(st.flops == p.flops);
      CHECK(st.kernel_calls >= 1);
      if (p.kernel != KernelKind::Elementwise) CHECK(st.kernel_calls == be.calls);
      std::int64_t nest = 1;
      for (const auto& l : p.loop_nest) nest *= l.extent;
      if (p.kernel != KernelKind::Dot || p.kernel_map.k2_label < 0) CHECK(st.kernel_calls == nest);
      const bool copies = p.kernel == KernelKind::CopyGemm || p.kernel == KernelKind::CopyGemv;
      if (!copies) CHECK(st.packed_bytes == 0);
      // workers do not change the result (include/tc/executor.hpp:25-27)
      const auto [res4, st4] = execute(p, b.v, b.left, b.right, be, 4);
      CHECK(std::memcmp(res.data(), res4.data(), static_cast<std::size_t>(res.size()) * 8) == 0);
      CHECK(st4.kernel_calls == st.kernel_calls);
    }
  }
}

TEST_CASE("a failing backend's error carries the slice coordinates") {  // test_executor.cpp:240-291
  const auto b = bind_expr("C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]",
                           {{"i", 4}, {"j", 4}, {"k", 3}, {"l", 5}});
  const ExecutionPlan p = plan(b.v);  // class 3.2: GEMM per l slice
  FailingBlas be(2);
  try {
    execute(p, b.v, b.left, b.right, be);
    CHECK(false);
  } catch (const std::runtime_error& e) {
    CHECK(std::string(e.what()) == "injected backend failure at slice coordinates [l=2]");
  }
  // the same through a worker pool: the first error propagates
  FailingBlas be2(0);
  CHECK_THROWS_AS(execute(p, b.v, b.left, b.right, be2, 3), std::runtime_error);
}

TEST_CASE("execute_into with a caller's backend fills caller storage") {
  const auto b = bind_expr("C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]",
                           {{"a", 3}, {"b", 4}, {"c", 2}, {"k", 5}});
  HostBlas be;
  const ExecutionPlan p = plan(b.v);
  std::vector<double> out(24, 7.0);  // overwritten whole
  const ExecutionStats st = execute_into(p, b.v, b.left.data(), b.right.data(), out.data(), be);
  const auto want = brute(b);
  double worst = 0;
  for (std::size_t i = 0; i < want.size(); ++i) worst = std::max(worst, std::fabs(out[i] - want[i]));
  CHECK(worst <= 1e-13);
  CHECK(st.kernel_calls == 2);  // one GEMM per c slice
}

// ------------------------------------------------------ metric (tc/metric.hpp)
// Restated from the reference's tests/test_metric.cpp; the contractions run
// slice by slice through the host test backend (no device in this suite).
namespace {
Tensor diagonal(std::initializer_list<double> d) {
  const auto n = static_cast<std::int64_t>(d.size());
  Tensor g = Tensor::zeros({n, n}, {Variance::Down, Variance::Down}, "g");
  std::int64_t i = 0;
  for (double x : d) g.data()[(i++) * (n + 1)] = x;
  return g;
}
const std::vector<double> kDense3{4, 1, 0.5, 1, 3, 0.25, 0.5, 0.25, 2};
bool near(double a, double b, double tol = 1e-12) { return std::fabs(a - b) <= tol * std::max(1.0, std::fabs(b)); }
}  // namespace

TEST_CASE("invert_metric: identity, diagonal, dense symmetric") {  // test_metric.cpp:28-60
  const auto id = invert_metric(diagonal({1, 1, 1}));
  CHECK(id.dimension == 3);
  for (int i = 0; i < 3; ++i) CHECK(id.g_inv.at({i, i}) == 1.0);
  const auto m = invert_metric(diagonal({1, 4, 4}));
  CHECK(near(m.g_inv.at({0, 0}), 1.0));
  CHECK(near(m.g_inv.at({1, 1}), 0.25));
  CHECK(near(m.g_inv.at({2, 2}), 0.25));
  CHECK(m.g_inv.at({0, 1}) == 0.0);
  CHECK(m.g_inv.variance(0) == Variance::Up);
  CHECK(m.g.variance(1) == Variance::Down);

  const auto d = invert_metric(
      Tensor::from_values({3, 3}, {Variance::Down, Variance::Down}, kDense3));
  for (std::int64_t i = 0; i < 3; ++i)
    for (std::int64_t j = 0; j < 3; ++j) {
      double acc = 0;
      for (std::int64_t k = 0; k < 3; ++k) acc += d.g.at({i, k}) * d.g_inv.at({k, j});
      CHECK(near(acc, i == j ? 1.0 : 0.0, 1e-14));
    }
  // a larger ill-scaled but regular case: pivoting must pick the big entries
  const std::int64_t n = 6;
  Tensor g = Tensor::zeros({n, n}, {Variance::Down, Variance::Down});
  for (std::int64_t i = 0; i < n; ++i)
    for (std::int64_t j = 0; j < n; ++j)
      g.data()[i + j * n] = (i == j ? 1e-3 * static_cast<double>(i + 1) : 0.0) +
                            1.0 / static_cast<double>(1 + i + j);
  const auto h = invert_metric(g);
  for (std::int64_t i = 0; i < n; ++i)
    for (std::int64_t j = 0; j < n; ++j) {
      double acc = 0;
      for (std::int64_t k = 0; k < n; ++k) acc += h.g.at({i, k}) * h.g_inv.at({k, j});
      CHECK(near(acc, i == j ? 1.0 : 0.0, 1e-9));
    }
}

TEST_CASE("invert_metric rejects bad input with the reference's messages") {  // :39-47
  Tensor g = diagonal({1, 2, 3});
  g.at({0, 1}) = 0.5;
  CHECK_THROWS_WITH_AS(invert_metric(g), "metric is not symmetric", std::invalid_argument);
  CHECK_THROWS_WITH_AS(invert_metric(diagonal({1, 0, 1})), "metric is singular",
                       std::invalid_argument);
  CHECK_THROWS_WITH_AS(invert_metric(Tensor::zeros({2, 3}, {Variance::Down, Variance::Down})),
                       "metric must be a square rank-2 tensor", std::invalid_argument);
  CHECK_THROWS_AS(invert_metric(diagonal({1.0, 1e-30, 1.0})), std::invalid_argument);
  CHECK_THROWS_WITH_AS(invert_metric(diagonal({1.0, 1e-13, 1.0})),
                       "metric is numerically singular", std::invalid_argument);
}

TEST_CASE("spherical metric values and singular points") {  // :62-76
  const auto unit = spherical_metric(1.0, M_PI / 2);
  for (int i = 0; i < 3; ++i) CHECK(near(unit.g.at({i, i}), 1.0));
  const auto m = spherical_metric(2.0, M_PI / 2);
  CHECK(near(m.g.at({1, 1}), 4.0));
  CHECK(near(m.g.at({2, 2}), 4.0));
  CHECK(near(m.g_inv.at({2, 2}), 0.25));
  CHECK(near(spherical_metric(2.0, M_PI / 6).g.at({2, 2}), 1.0));
  CHECK_THROWS_AS(spherical_metric(0.0, 1.0), std::invalid_argument);
  CHECK_THROWS_AS(spherical_metric(1.0, 0.0), std::invalid_argument);
}

TEST_CASE("lowering and raising through a caller's backend") {  // :78-151
  HostBlas be;
  const auto id = invert_metric(diagonal({1, 1, 1}));
  const Tensor t = Tensor::seeded_random({3, 3}, {Variance::Up, Variance::Up}, 3);
  const Tensor low = lower_index(t, 1, id, be);
  CHECK(low.variance(1) == Variance::Down);
  CHECK(low.variance(0) == Variance::Up);
  for (std::int64_t i = 0; i < t.size(); ++i) CHECK(near(low.data()[i], t.data()[i], 1e-14));
  CHECK(be.calls > 0);

  const auto sph = spherical_metric(2.0, M_PI / 2);
  const Tensor v = Tensor::from_values({3}, {Variance::Up}, {1, 1, 1}, "v");
  const Tensor lv = lower_index(v, 0, sph, be);
  CHECK(near(lv.at({0}), 1.0));
  CHECK(near(lv.at({1}), 4.0));
  CHECK(near(lv.at({2}), 4.0));
  const Tensor back = raise_index(lv, 0, invert_metric(diagonal({1, 4, 4})), be);
  for (int i = 0; i < 3; ++i) CHECK(near(back.at({i}), 1.0));

  const auto dense = invert_metric(
      Tensor::from_values({3, 3}, {Variance::Down, Variance::Down}, kDense3));
  const Tensor w =
      Tensor::seeded_random({3, 4, 3}, {Variance::Up, Variance::Down, Variance::Up}, 5);
  for (const int mode : {0, 2}) {
    const Tensor rt = raise_index(lower_index(w, mode, dense, be), mode, dense, be);
    CHECK(max_rel_error(rt, w) <= 1e-10);
  }
  // lowering distinct modes commutes
  const auto m2 = invert_metric(
      Tensor::from_values({2, 2}, {Variance::Down, Variance::Down}, {2, 0.5, 0.5, 3}));
  const Tensor c = Tensor::seeded_random({2, 2, 2}, std::vector<Variance>(3, Variance::Up), 9);
  CHECK(max_rel_error(lower_index(lower_index(c, 0, m2, be), 2, m2, be),
                      lower_index(lower_index(c, 2, m2, be), 0, m2, be)) <= 1e-12);
}

TEST_CASE("metric variance, extent and mode guards") {  // :134-142, src/metric.cpp:64-70
  HostBlas be;
  const auto m = spherical_metric(2.0, 1.0);
  CHECK_THROWS_WITH_AS(lower_index(Tensor::zeros({3}, {Variance::Down}), 0, m, be),
                       "mode is already lowered", std::invalid_argument);
  CHECK_THROWS_WITH_AS(raise_index(Tensor::zeros({3}, {Variance::Up}), 0, m, be),
                       "mode is already raised", std::invalid_argument);
  CHECK_THROWS_WITH_AS(lower_index(Tensor::zeros({4}, {Variance::Up}), 0, m, be),
                       "mode extent does not match metric dimension", std::invalid_argument);
  CHECK_THROWS_WITH_AS(lower_index(Tensor::zeros({3}, {Variance::Up}), 1, m, be),
                       "mode out of range", std::invalid_argument);
}

TEST_CASE("metrics serialize through the tensor text format") {  // :220-226
  const auto m = spherical_metric(2.0, M_PI / 3);
  std::stringstream ss;
  write_tensor(ss, m.g);
  CHECK(max_rel_error(read_tensor(ss), m.g) == 0.0);
}

TH_MAIN
