// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the *unmodified* reference library (tcontract, compiled by
// oracle/Makefile from /root/reference/proj/src into oracle/_ref/). It lets
// pytest and bench.py's CPU arms drive the reference through ctypes:
//   ref_report   parse → validate → classify/enumerate/plan/render  (text)
//   ref_execute  tc::execute with the reference CPU backend
//   ref_naive    tc::contract_naive (brute-force oracle)
//   ref_seeded   tc::Tensor::seeded_random
//   ref_gemm     ReferenceBackend::gemm on caller buffers
// The same report format is produced by the product front (tcf_report in
// paper_1307_2100_b200/csrc/host/capi_front.cpp) so the two can be diffed.
#include <cstdint>
#include <cstring>
#include <map>
#include <sstream>
#include <string>

#include "tc/executor.hpp"
#include "tc/tensor_io.hpp"
#include "tc/oracle.hpp"
#include "tc/planner.hpp"

namespace {

std::map<std::string, std::int64_t> extents_of(const char* s) {
  std::map<std::string, std::int64_t> out;
  std::istringstream is(s ? s : "");
  std::string item;
  while (std::getline(is, item, ',')) {
    if (item.empty()) continue;
    const auto eq = item.find('=');
    if (eq == std::string::npos) throw tc::parse_error("bad extents", 0);
    out[item.substr(0, eq)] = std::stoll(item.substr(eq + 1));
  }
  return out;
}

tc::Tensor operand(const tc::TensorExpr& te, const std::map<std::string, std::int64_t>& ext,
                   std::uint64_t seed) {
  std::vector<std::int64_t> e;
  std::vector<tc::Variance> v;
  for (const auto& idx : te.indices) {
    e.push_back(ext.at(idx.label));
    v.push_back(idx.var);
  }
  return tc::Tensor::seeded_random(e, v, seed, te.name);
}

struct Bound {
  tc::ContractionSpec spec;
  tc::Tensor left, right;
  tc::ValidatedContraction v;
};

Bound bind(const char* expr, int positional, const char* extents, std::uint64_t seed) {
  Bound b;
  b.spec = tc::parse(expr, positional != 0);
  const auto ext = extents_of(extents);
  b.left = operand(b.spec.left, ext, seed);
  b.right = operand(b.spec.right, ext, seed + 1);
  b.v = tc::validate(b.spec, b.left, b.right);
  return b;
}

std::string vec(const tc::SlicingVector& s) {
  std::string t = "(";
  for (std::size_t i = 0; i < s.size(); ++i) {
    if (i) t += ' ';
    t += s[i] ? '1' : '0';
  }
  return t + ")";
}

tc::SlicingVector parse_vec(const char* s) {
  tc::SlicingVector v;
  for (const char* p = s; p && *p; ++p)
    if (*p == '0' || *p == '1') v.push_back(static_cast<std::uint8_t>(*p - '0'));
  return v;
}

std::string report(const Bound& b) {
  const auto& v = b.v;
  std::ostringstream os;
  os << "spec: " << tc::unparse(b.spec) << "\n";
  os << "labels:";
  for (const auto& l : v.labels)
    os << ' ' << l.label << ':' << l.extent << ':' << l.left_mode << ':' << l.right_mode << ':'
       << l.output_mode << ':' << (l.contracted ? 'c' : 'f');
  os << "\ncontracted:";
  for (int i : v.contracted) os << ' ' << i;
  os << "\nleft_free:";
  for (int i : v.left_free) os << ' ' << i;
  os << "\nright_free:";
  for (int i : v.right_free) os << ' ' << i;
  os << "\np: " << v.p << " delta: " << v.delta_left << ' ' << v.delta_right << "\n";
  os << "class: " << tc::to_string(tc::classify(v)) << "\n";
  os << "flops: " << tc::flop_count(v) << "\n";
  os << "options:\n";
  for (const auto& o : tc::enumerate_slicings(v))
    os << vec(o.s_left) << '|' << vec(o.s_right) << '|' << o.report.r1_ok << o.report.r2_ok
       << o.report.r3_ok << '|' << tc::to_string(o.report.fallback) << '|'
       << tc::to_string(o.report.kernel) << '|' << o.kernel_dims_product << '|'
       << o.output_staged << "\n";
  os << "auto:\n";
  try {
    const auto p = tc::plan(v);
    os << tc::render_plan(p, v);
    os << "loop_extents:";
    for (const auto& l : p.loop_nest) os << ' ' << l.extent;
    os << "\nkm: " << p.kernel_map.a_is_left << p.kernel_map.matrix_is_left << "\n";
  } catch (const std::exception& e) {
    os << "error: " << e.what() << "\n";
  }
  for (int k = 0; k <= static_cast<int>(tc::KernelKind::Elementwise); ++k) {
    const auto kind = static_cast<tc::KernelKind>(k);
    os << "force " << tc::to_string(kind) << ":\n";
    try {
      const auto p = tc::plan(v, tc::PlanPolicy::force_kernel(kind));
      os << tc::render_plan(p, v);
    } catch (const std::exception& e) {
      os << "error: " << e.what() << "\n";
    }
  }
  const auto adv = tc::relayout_advice(v);
  os << "relayout: " << (adv ? *adv : std::string("none")) << "\n";
  return os.str();
}

int fail(const std::exception& e, char* buf, std::int64_t cap, int code) {
  if (buf && cap > 0) {
    std::strncpy(buf, e.what(), static_cast<std::size_t>(cap - 1));
    buf[cap - 1] = 0;
  }
  return code;
}

int put(const std::string& s, char* buf, std::int64_t cap) {
  if (static_cast<std::int64_t>(s.size()) + 1 > cap) return 4;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return 0;
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) int ref_report(const char* expr, int positional,
                                                      const char* extents, char* buf,
                                                      std::int64_t cap) {
  try {
    return put(report(bind(expr, positional, extents, 1)), buf, cap);
  } catch (const tc::parse_error& e) {
    return fail(e, buf, cap, 2);
  } catch (const std::exception& e) {
    return fail(e, buf, cap, 1);
  }
}

// policy: 0 auto, 1 force kernel (kernel = KernelKind index), 2 force slicing.
// stats: kernel_calls, packed_bytes, staged_bytes, flops; *seconds = wall.
__attribute__((visibility("default"))) int ref_execute(
    const char* expr, int positional, const char* extents, std::uint64_t seed, int workers,
    int policy, int kernel, const char* sl, const char* sr, double* out, std::int64_t out_cap,
    std::int64_t* stats, double* seconds, char* err, std::int64_t errcap) {
  try {
    const Bound b = bind(expr, positional, extents, seed);
    tc::PlanPolicy pol;
    if (policy == 1) pol = tc::PlanPolicy::force_kernel(static_cast<tc::KernelKind>(kernel));
    if (policy == 2) pol = tc::PlanPolicy::force_slicing(parse_vec(sl), parse_vec(sr));
    const auto p = tc::plan(b.v, pol);
    const auto backend = tc::make_reference_backend();
    auto [res, st] = tc::execute(p, b.v, b.left, b.right, *backend, workers);
    if (res.size() > out_cap) throw std::invalid_argument("output buffer too small");
    std::memcpy(out, res.data(), static_cast<std::size_t>(res.size()) * 8);
    if (stats) {
      stats[0] = st.kernel_calls;
      stats[1] = st.packed_bytes;
      stats[2] = st.staged_bytes;
      stats[3] = st.flops;
    }
    if (seconds) *seconds = st.wall_seconds;
    return 0;
  } catch (const tc::parse_error& e) {
    return fail(e, err, errcap, 2);
  } catch (const tc::resource_limit_error& e) {
    return fail(e, err, errcap, 3);
  } catch (const std::exception& e) {
    return fail(e, err, errcap, 1);
  }
}

// Bound contraction for repeated timing (bench.py's reference arm): operands
// seeded and the plan built once by ref_bind; ref_run is one tc::execute
// (src/executor.cpp:287-369) with the reference backend, its wall time in
// *seconds (ExecutionStats::wall_seconds); `out` may be null.
struct RefBound {
  Bound b;
  tc::ExecutionPlan plan;
};

__attribute__((visibility("default"))) void* ref_bind(const char* expr, int positional,
                                                      const char* extents, std::uint64_t seed,
                                                      int policy, int kernel, const char* sl,
                                                      const char* sr, char* err,
                                                      std::int64_t errcap) {
  try {
    auto* h = new RefBound{bind(expr, positional, extents, seed), {}};
    tc::PlanPolicy pol;
    if (policy == 1) pol = tc::PlanPolicy::force_kernel(static_cast<tc::KernelKind>(kernel));
    if (policy == 2) pol = tc::PlanPolicy::force_slicing(parse_vec(sl), parse_vec(sr));
    try {
      h->plan = tc::plan(h->b.v, pol);
    } catch (...) {
      delete h;
      throw;
    }
    return h;
  } catch (const std::exception& e) {
    fail(e, err, errcap, 1);
    return nullptr;
  }
}

__attribute__((visibility("default"))) int ref_run(void* handle, int workers, double* out,
                                                   std::int64_t out_cap, std::int64_t* stats,
                                                   double* seconds, char* err,
                                                   std::int64_t errcap) {
  try {
    auto* h = static_cast<RefBound*>(handle);
    const auto backend = tc::make_reference_backend();
    auto [res, st] = tc::execute(h->plan, h->b.v, h->b.left, h->b.right, *backend, workers);
    if (out) {
      if (res.size() > out_cap) throw std::invalid_argument("output buffer too small");
      std::memcpy(out, res.data(), static_cast<std::size_t>(res.size()) * 8);
    }
    if (stats) {
      stats[0] = st.kernel_calls;
      stats[1] = st.packed_bytes;
      stats[2] = st.staged_bytes;
      stats[3] = st.flops;
    }
    if (seconds) *seconds = st.wall_seconds;
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errcap, 1);
  }
}

__attribute__((visibility("default"))) void ref_release(void* handle) {
  delete static_cast<RefBound*>(handle);
}

__attribute__((visibility("default"))) int ref_naive(const char* expr, int positional,
                                                     const char* extents, std::uint64_t seed,
                                                     std::int64_t work_cap, double* out,
                                                     std::int64_t out_cap, std::int64_t* macs,
                                                     char* err, std::int64_t errcap) {
  try {
    const Bound b = bind(expr, positional, extents, seed);
    tc::OracleStats st;
    const auto res = tc::contract_naive(b.v, b.left, b.right, work_cap, &st);
    if (res.size() > out_cap) throw std::invalid_argument("output buffer too small");
    std::memcpy(out, res.data(), static_cast<std::size_t>(res.size()) * 8);
    if (macs) *macs = st.multiply_adds;
    return 0;
  } catch (const tc::resource_limit_error& e) {
    return fail(e, err, errcap, 3);
  } catch (const std::exception& e) {
    return fail(e, err, errcap, 1);
  }
}

__attribute__((visibility("default"))) int ref_seeded(int rank, const std::int64_t* ext,
                                                      std::uint64_t seed, double* out) {
  try {
    std::vector<std::int64_t> e(ext, ext + rank);
    const auto t = tc::Tensor::seeded_random(e, std::vector<tc::Variance>(rank, tc::Variance::Up),
                                             seed);
    std::memcpy(out, t.data(), static_cast<std::size_t>(t.size()) * 8);
    return 0;
  } catch (...) {
    return 1;
  }
}

__attribute__((visibility("default"))) int ref_gemm(int ta, int tb, std::int64_t m,
                                                    std::int64_t n, std::int64_t k, double alpha,
                                                    const double* a, std::int64_t lda,
                                                    const double* b, std::int64_t ldb,
                                                    double beta, double* c, std::int64_t ldc,
                                                    char* err, std::int64_t errcap) {
  try {
    tc::make_reference_backend()->gemm(ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errcap, 1);
  }
}

// TENSOR v1 text of Tensor::seeded_random(ext, var, seed, name) through the
// reference writer (src/tensor_io.cpp:11-27); 4 = buffer too small.
__attribute__((visibility("default"))) int ref_tensor_text(const std::int64_t* ext, int rank,
                                                           const char* var, std::uint64_t seed,
                                                           const char* name, char* buf,
                                                           std::int64_t cap) {
  try {
    std::vector<std::int64_t> e(ext, ext + rank);
    std::vector<tc::Variance> v;
    for (int i = 0; i < rank; ++i) v.push_back(var[i] == '-' ? tc::Variance::Down : tc::Variance::Up);
    const tc::Tensor t = tc::Tensor::seeded_random(std::move(e), std::move(v), seed, name);
    std::ostringstream os;
    tc::write_tensor(os, t);
    return put(os.str(), buf, cap);
  } catch (const std::exception& e) {
    return fail(e, buf, cap, 1);
  }
}

// Parse TENSOR v1 text with the reference reader (src/tensor_io.cpp:53-85):
// values into out (cap elements), *n = element count; errors as messages.
__attribute__((visibility("default"))) int ref_read_tensor_text(const char* text, double* out,
                                                                std::int64_t cap,
                                                                std::int64_t* n, char* err,
                                                                std::int64_t errcap) {
  try {
    std::istringstream is(text ? text : "");
    const tc::Tensor t = tc::read_tensor(is);
    *n = t.size();
    if (t.size() > cap) throw std::invalid_argument("output buffer too small");
    std::memcpy(out, t.data(), static_cast<std::size_t>(t.size()) * 8);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errcap, 1);
  }
}

}  // extern "C"
