// Plan-level C-ABI (include/tcf.h) over the tc:: front. Host C++ only.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <sstream>
#include <string>

#include "tc/metric.hpp"
#include "tc/contract.hpp"
#include "tcb.h"
#include "tcf.h"

namespace {

thread_local std::string g_err;

std::map<std::string, std::int64_t> parse_extents(const char* s) {
  // "label=N,label=N" (the CLI's --extents, tools/tcontract.cpp:23-36)
  std::map<std::string, std::int64_t> out;
  std::istringstream is(s ? s : "");
  std::string item;
  while (std::getline(is, item, ',')) {
    if (item.empty()) continue;
    const auto eq = item.find('=');
    if (eq == std::string::npos) throw tc::parse_error("--extents entries must look like label=N", 0);
    const std::int64_t value = std::stoll(item.substr(eq + 1));
    if (value <= 0) throw tc::parse_error("extent must be positive", 0);
    out[item.substr(0, eq)] = value;
  }
  return out;
}

struct Shapes {
  std::vector<std::int64_t> le, re;
  std::vector<tc::Variance> lv, rv;
};

Shapes shapes_of(const tc::ContractionSpec& spec, const std::map<std::string, std::int64_t>& ext) {
  Shapes s;
  auto fill = [&](const tc::TensorExpr& t, std::vector<std::int64_t>& e,
                  std::vector<tc::Variance>& v) {
    for (const auto& ix : t.indices) {
      const auto it = ext.find(ix.label);
      if (it == ext.end()) throw tc::parse_error("no extent given for label '" + ix.label + "'", 0);
      e.push_back(it->second);
      v.push_back(ix.var);
    }
  };
  fill(spec.left, s.le, s.lv);
  fill(spec.right, s.re, s.rv);
  return s;
}

std::string vec_text(const tc::SlicingVector& s) {
  std::string t = "(";
  for (std::size_t i = 0; i < s.size(); ++i) {
    if (i) t += ' ';
    t += s[i] ? '1' : '0';
  }
  return t + ")";
}

tc::SlicingVector vec_parse(const char* s) {
  tc::SlicingVector v;
  for (const char* p = s; p && *p; ++p)
    if (*p == '0' || *p == '1') v.push_back(static_cast<std::uint8_t>(*p - '0'));
  return v;
}

std::string report(const tc::ValidatedContraction& v) {
  std::ostringstream os;
  os << "spec: " << tc::unparse(v.spec) << "\nlabels:";
  for (const auto& l : v.labels)
    os << ' ' << l.label << ':' << l.extent << ':' << l.left_mode << ':' << l.right_mode << ':'
       << l.output_mode << ':' << (l.contracted ? 'c' : 'f');
  auto ids = [&](const char* tag, const std::vector<int>& xs) {
    os << '\n' << tag << ':';
    for (int x : xs) os << ' ' << x;
  };
  ids("contracted", v.contracted);
  ids("left_free", v.left_free);
  ids("right_free", v.right_free);
  os << "\np: " << v.p << " delta: " << v.delta_left << ' ' << v.delta_right << '\n'
     << "class: " << tc::to_string(tc::classify(v)) << '\n'
     << "flops: " << tc::flop_count(v) << "\noptions:\n";
  for (const auto& o : tc::enumerate_slicings(v))
    os << vec_text(o.s_left) << '|' << vec_text(o.s_right) << '|' << o.report.r1_ok
       << o.report.r2_ok << o.report.r3_ok << '|' << tc::to_string(o.report.fallback) << '|'
       << tc::to_string(o.report.kernel) << '|' << o.kernel_dims_product << '|'
       << o.output_staged << '\n';
  os << "auto:\n";
  try {
    const tc::ExecutionPlan p = tc::plan(v);
    os << tc::render_plan(p, v) << "loop_extents:";
    for (const auto& l : p.loop_nest) os << ' ' << l.extent;
    os << "\nkm: " << p.kernel_map.a_is_left << p.kernel_map.matrix_is_left << '\n';
  } catch (const std::exception& e) {
    os << "error: " << e.what() << '\n';
  }
  for (int k = 0; k <= static_cast<int>(tc::KernelKind::Elementwise); ++k) {
    const auto kind = static_cast<tc::KernelKind>(k);
    os << "force " << tc::to_string(kind) << ":\n";
    try {
      os << tc::render_plan(tc::plan(v, tc::PlanPolicy::force_kernel(kind)), v);
    } catch (const std::exception& e) {
      os << "error: " << e.what() << '\n';
    }
  }
  const auto adv = tc::relayout_advice(v);
  os << "relayout: " << (adv ? *adv : std::string("none")) << '\n';
  return os.str();
}

int fail(const std::exception& e, int code, char* err, std::int64_t cap) {
  g_err = e.what();
  if (err && cap > 0) {
    std::strncpy(err, e.what(), static_cast<std::size_t>(cap - 1));
    err[cap - 1] = 0;
  }
  return code;
}

#define TCF_GUARD(err, cap)                                      \
  catch (const tc::parse_error& e) { return fail(e, 2, err, cap); } \
  catch (const tc::resource_limit_error& e) { return fail(e, 3, err, cap); } \
  catch (const std::exception& e) { return fail(e, 1, err, cap); }

struct Handle {
  tc::ValidatedContraction v;
  std::unique_ptr<tc::PreparedContraction> pc;
  int device = 0;
  std::int32_t path = -1;
};

}  // namespace

extern "C" {

const char* tcf_last_error(void) { return g_err.c_str(); }

int tcf_report(const char* expr, int positional, const char* extents, char* buf, int64_t cap) {
  try {
    const tc::ContractionSpec spec = tc::parse(expr ? expr : "", positional != 0);
    const Shapes s = shapes_of(spec, parse_extents(extents));
    const std::string text = report(tc::validate_shapes(spec, s.le, s.lv, s.re, s.rv));
    if (static_cast<std::int64_t>(text.size()) + 1 > cap) return 4;
    std::memcpy(buf, text.c_str(), text.size() + 1);
    return 0;
  }
  TCF_GUARD(buf, cap)
}

int tcf_execute(const char* expr, int positional, const char* extents, uint64_t seed,
                int workers, int policy, int kernel, const char* s_left, const char* s_right,
                double* out, int64_t out_cap, int64_t* stats, double* seconds, char* err,
                int64_t errcap) {
  try {
    const tc::ContractionSpec spec = tc::parse(expr ? expr : "", positional != 0);
    const Shapes s = shapes_of(spec, parse_extents(extents));
    const tc::Tensor left = tc::Tensor::seeded_random(s.le, s.lv, seed, spec.left.name);
    const tc::Tensor right = tc::Tensor::seeded_random(s.re, s.rv, seed + 1, spec.right.name);
    const tc::ValidatedContraction v = tc::validate(spec, left, right);
    tc::PlanPolicy pol;
    if (policy == 1) pol = tc::PlanPolicy::force_kernel(static_cast<tc::KernelKind>(kernel));
    if (policy == 2) pol = tc::PlanPolicy::force_slicing(vec_parse(s_left), vec_parse(s_right));
    const tc::ExecutionPlan p = tc::plan(v, pol);
    const auto backend = tc::make_b200_backend();
    auto [res, st] = tc::execute(p, v, left, right, *backend, workers);
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
  }
  TCF_GUARD(err, errcap)
}

int tcf_execute_host(const char* expr, int positional, const char* extents, const double* left,
                     const double* right, double* out, int64_t out_cap, int workers, int policy,
                     int kernel, const char* s_left, const char* s_right, int64_t* stats,
                     double* seconds, char* err, int64_t errcap) {
  try {
    static const bool trace = std::getenv("TC_EXEC_TRACE") != nullptr;  // diagnostics
    const auto t0 = std::chrono::steady_clock::now();
    const tc::ContractionSpec spec = tc::parse(expr ? expr : "", positional != 0);
    const Shapes s = shapes_of(spec, parse_extents(extents));
    const tc::ValidatedContraction v = tc::validate_shapes(spec, s.le, s.lv, s.re, s.rv);
    std::int64_t n = 1;
    for (std::int64_t e : v.output_extents()) n *= e;
    if (n > out_cap) throw std::invalid_argument("output buffer too small");
    if (!left || !right || !out) throw std::invalid_argument("null operand or result buffer");
    tc::PlanPolicy pol;
    if (policy == 1) pol = tc::PlanPolicy::force_kernel(static_cast<tc::KernelKind>(kernel));
    if (policy == 2) pol = tc::PlanPolicy::force_slicing(vec_parse(s_left), vec_parse(s_right));
    const tc::ExecutionPlan p = tc::plan(v, pol);
    if (trace)
      std::fprintf(stderr, "front parse+plan %8.3f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                       .count());
    static const auto backend = tc::make_b200_backend();
    const tc::ExecutionStats st = tc::execute_into(p, v, left, right, out, *backend, workers);
    if (trace)
      std::fprintf(stderr, "front returned   %8.3f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                       .count());
    if (stats) {
      stats[0] = st.kernel_calls;
      stats[1] = st.packed_bytes;
      stats[2] = st.staged_bytes;
      stats[3] = st.flops;
    }
    if (seconds) *seconds = st.wall_seconds;
    return 0;
  }
  TCF_GUARD(err, errcap)
}

int tcf_contract_naive(const char* expr, int positional, const char* extents, uint64_t seed,
                       int64_t work_cap, double* out, int64_t out_cap, int64_t* macs, char* err,
                       int64_t errcap) {
  try {
    const tc::ContractionSpec spec = tc::parse(expr ? expr : "", positional != 0);
    const Shapes s = shapes_of(spec, parse_extents(extents));
    const tc::Tensor left = tc::Tensor::seeded_random(s.le, s.lv, seed, spec.left.name);
    const tc::Tensor right = tc::Tensor::seeded_random(s.re, s.rv, seed + 1, spec.right.name);
    const tc::ValidatedContraction v = tc::validate(spec, left, right);
    tc::OracleStats st;
    const tc::Tensor res = tc::contract_naive(v, left, right, work_cap, &st);
    if (res.size() > out_cap) throw std::invalid_argument("output buffer too small");
    std::memcpy(out, res.data(), static_cast<std::size_t>(res.size()) * 8);
    if (macs) *macs = st.multiply_adds;
    return 0;
  }
  TCF_GUARD(err, errcap)
}

int tcf_lower(const char* expr, int positional, const char* extents, char* buf, int64_t cap) {
  try {
    const tc::ContractionSpec spec = tc::parse(expr ? expr : "", positional != 0);
    const Shapes s = shapes_of(spec, parse_extents(extents));
    const std::string text = tc::lower(tc::validate_shapes(spec, s.le, s.lv, s.re, s.rv)).summary();
    if (static_cast<std::int64_t>(text.size()) + 1 > cap) return 4;
    std::memcpy(buf, text.c_str(), text.size() + 1);
    return 0;
  }
  TCF_GUARD(buf, cap)
}

int tcf_seeded(int64_t n, uint64_t seed, double* out) {
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (int64_t i = 0; i < n; ++i) out[i] = u(gen);
  return 0;
}

int tcf_seeded_block(uint64_t seed, int rank, const int64_t* ext, int mode, int64_t lo,
                     int64_t hi, double* out) {
  if (rank < 1 || mode < 0 || mode >= rank || !ext || !out) {
    g_err = "tcf_seeded_block: bad arguments";
    return 1;
  }
  int64_t below = 1, outer = 1;
  for (int m = 0; m < mode; ++m) below *= ext[m];
  for (int m = mode + 1; m < rank; ++m) outer *= ext[m];
  const int64_t e = ext[mode];
  if (lo < 0 || hi > e || lo >= hi) {
    g_err = "tcf_seeded_block: empty or out-of-range block";
    return 1;
  }
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);  // one draw per value
  double* o = out;
  for (int64_t q = 0; q < outer; ++q) {
    gen.discard(static_cast<unsigned long long>(below * lo));
    for (int64_t i = 0; i < below * (hi - lo); ++i) *o++ = u(gen);
    if (q + 1 < outer) gen.discard(static_cast<unsigned long long>(below * (e - hi)));
  }
  return 0;
}

int tcf_prepare(const char* expr, int positional, const char* extents, int device, void** handle,
                char* err, int64_t errcap) {
  try {
    auto h = std::make_unique<Handle>();
    const tc::ContractionSpec spec = tc::parse(expr ? expr : "", positional != 0);
    const Shapes s = shapes_of(spec, parse_extents(extents));
    h->v = tc::validate_shapes(spec, s.le, s.lv, s.re, s.rv);
    h->device = device;
    h->pc = std::make_unique<tc::PreparedContraction>(h->v, device);
    *handle = h.release();
    return 0;
  }
  TCF_GUARD(err, errcap)
}

int tcf_upload(void* handle, const double* left, const double* right) {
  try {
    static_cast<Handle*>(handle)->pc->upload(left, right);
    return 0;
  }
  TCF_GUARD(nullptr, 0)
}

int tcf_run(void* handle) {
  try {
    Handle* h = static_cast<Handle*>(handle);
    h->pc->run();
    tcb_gemm_info info{};
    tcb_last_gemm_info(&info);
    h->path = info.path;
    return 0;
  }
  TCF_GUARD(nullptr, 0)
}

int tcf_run_permutes(void* handle) {
  try {
    static_cast<Handle*>(handle)->pc->run_permutes();
    return 0;
  }
  TCF_GUARD(nullptr, 0)
}

int tcf_run_contraction(void* handle) {
  try {
    Handle* h = static_cast<Handle*>(handle);
    h->pc->run_contraction();
    tcb_gemm_info info{};
    tcb_last_gemm_info(&info);
    h->path = info.path;
    return 0;
  }
  TCF_GUARD(nullptr, 0)
}

int tcf_run_scattered(void* handle, double* base, int parts, int64_t part_stride) {
  try {
    Handle* h = static_cast<Handle*>(handle);
    h->pc->run_scattered(base, parts, part_stride);
    tcb_gemm_info info{};
    tcb_last_gemm_info(&info);
    h->path = info.path;
    return 0;
  }
  TCF_GUARD(nullptr, 0)
}

int tcf_run_streamed(void* handle, const double* left, const double* right, double* out,
                     int slabs, int* slabs_used) {
  try {
    const int n = static_cast<Handle*>(handle)->pc->run_streamed(left, right, out, slabs);
    if (slabs_used) *slabs_used = n;
    return 0;
  }
  TCF_GUARD(nullptr, 0)
}

int tcf_run_streamed_async(void* handle, const double* left, const double* right, double* out,
                           int slabs, int* slabs_used) {
  try {
    const int n =
        static_cast<Handle*>(handle)->pc->run_streamed(left, right, out, slabs, /*wait=*/false);
    if (slabs_used) *slabs_used = n;
    return 0;
  }
  TCF_GUARD(nullptr, 0)
}

int tcf_download(void* handle, double* out) {
  try {
    static_cast<Handle*>(handle)->pc->download(out);
    return 0;
  }
  TCF_GUARD(nullptr, 0)
}

int tcf_sync(void* handle) {
  try {
    static_cast<Handle*>(handle)->pc->sync();
    return 0;
  }
  TCF_GUARD(nullptr, 0)
}

int tcf_info(void* handle, int64_t* info, char* summary, int64_t cap) {
  try {
    const Handle* h = static_cast<const Handle*>(handle);
    const tc::PreparedContraction& pc = *h->pc;
    const tc::DeviceRecipe& r = pc.recipe();
    std::int64_t batch = 1;
    for (std::int64_t e : r.bat_ext) batch *= e;
    const std::int64_t vals[12] = {pc.left_elements(),  pc.right_elements(), pc.output_elements(),
                                   pc.launches_last_run(), pc.permuted_bytes(), r.m,
                                   r.n,                 r.k,                batch,
                                   tc::flop_count(h->v), static_cast<std::int64_t>(r.permutes.size()),
                                   h->path};
    if (info) std::memcpy(info, vals, sizeof vals);
    if (summary && cap > 0) {
      const std::string s = r.summary();
      std::strncpy(summary, s.c_str(), static_cast<std::size_t>(cap - 1));
      summary[cap - 1] = 0;
    }
    return 0;
  }
  TCF_GUARD(nullptr, 0)
}

int tcf_device_ptrs(void* handle, void** left, void** right, void** out) {
  const Handle* h = static_cast<const Handle*>(handle);
  if (left) *left = h->pc->left_device();
  if (right) *right = h->pc->right_device();
  if (out) *out = h->pc->output_device();
  return 0;
}

int tcf_release(void* handle) {
  try {
    delete static_cast<Handle*>(handle);
    return 0;
  }
  TCF_GUARD(nullptr, 0)
}

int tcf_tensor_text(const int64_t* ext, int rank, const char* var, uint64_t seed,
                    const char* name, char* buf, int64_t cap) {
  try {
    if (rank < 0 || (rank > 0 && (!ext || !var))) throw std::invalid_argument("bad tensor shape");
    std::vector<std::int64_t> e(ext, ext + rank);
    std::vector<tc::Variance> v;
    for (int i = 0; i < rank; ++i) v.push_back(var[i] == '-' ? tc::Variance::Down : tc::Variance::Up);
    const tc::Tensor t = tc::Tensor::seeded_random(std::move(e), std::move(v), seed, name ? name : "");
    std::ostringstream os;
    tc::write_tensor(os, t);
    const std::string text = os.str();
    if (static_cast<std::int64_t>(text.size()) + 1 > cap) return 4;
    std::memcpy(buf, text.c_str(), text.size() + 1);
    return 0;
  }
  TCF_GUARD(buf, cap)
}

int tcf_read_tensor_text(const char* text, double* out, int64_t cap, int64_t* n, char* err,
                         int64_t errcap) {
  try {
    std::istringstream is(text ? text : "");
    const tc::Tensor t = tc::read_tensor(is);
    if (n) *n = t.size();
    if (t.size() > cap) return 4;
    std::memcpy(out, t.data(), static_cast<std::size_t>(t.size()) * 8);
    return 0;
  }
  TCF_GUARD(err, errcap)
}

int tcf_invert_metric(int64_t n, const double* g, double* g_inv, char* err, int64_t errcap) {
  try {
    if (n < 0 || !g || !g_inv) throw std::invalid_argument("bad metric buffers");
    tc::Tensor G = tc::Tensor::zeros({n, n}, {tc::Variance::Down, tc::Variance::Down}, "g");
    std::memcpy(G.data(), g, static_cast<std::size_t>(n * n) * 8);
    const tc::MetricTensor m = tc::invert_metric(G);
    std::memcpy(g_inv, m.g_inv.data(), static_cast<std::size_t>(n * n) * 8);
    return 0;
  }
  TCF_GUARD(err, errcap)
}

int tcf_metric_apply(const int64_t* ext, int rank, const char* var, const double* t, int mode,
                     int64_t n, const double* g, int raise, double* out, int64_t out_cap,
                     char* err, int64_t errcap) {
  try {
    if (rank < 0 || (rank > 0 && (!ext || !var)) || !t || !g || !out)
      throw std::invalid_argument("bad tensor shape");
    std::vector<std::int64_t> e(ext, ext + rank);
    std::vector<tc::Variance> v;
    for (int i = 0; i < rank; ++i) v.push_back(var[i] == '-' ? tc::Variance::Down : tc::Variance::Up);
    tc::Tensor T = tc::Tensor::zeros(std::move(e), std::move(v), "t");
    std::memcpy(T.data(), t, static_cast<std::size_t>(T.size()) * 8);
    tc::Tensor G = tc::Tensor::zeros({n, n}, {tc::Variance::Down, tc::Variance::Down}, "g");
    std::memcpy(G.data(), g, static_cast<std::size_t>(n * n) * 8);
    const tc::MetricTensor m = tc::invert_metric(G);
    const auto backend = tc::make_backend("b200");
    const tc::Tensor r = raise ? tc::raise_index(T, mode, m, *backend)
                               : tc::lower_index(T, mode, m, *backend);
    if (r.size() > out_cap) return 4;
    std::memcpy(out, r.data(), static_cast<std::size_t>(r.size()) * 8);
    return 0;
  }
  TCF_GUARD(err, errcap)
}

int tcf_bench_csv(const char* experiment, const char* sizes, const char* kernels,
                  const char* backend, int repetitions, uint64_t seed, int verify, int workers,
                  const char* custom_expr, const char* custom_extents, char* csv, int64_t cap,
                  int* verified) {
  try {
    tc::BenchConfig cfg;
    cfg.experiment = experiment ? experiment : "square3d";
    {
      std::istringstream is(sizes ? sizes : "");
      for (std::string item; std::getline(is, item, ',');)
        if (!item.empty()) cfg.sizes.push_back(std::stoll(item));
    }
    {
      std::istringstream is(kernels ? kernels : "");
      for (std::string item; std::getline(is, item, ',');) {
        if (item.empty()) continue;
        const auto k = tc::kernel_from_string(item);
        if (!k) throw std::invalid_argument("unknown kernel '" + item + "'");
        cfg.kernels.push_back(*k);
      }
    }
    if (backend && *backend) cfg.backend = backend;
    cfg.repetitions = repetitions;
    cfg.seed = seed;
    cfg.verify_sample = verify != 0;
    cfg.workers = workers;
    if (custom_expr) cfg.custom_expr = custom_expr;
    cfg.custom_extents = parse_extents(custom_extents);
    const auto rows = tc::run_bench(cfg);
    std::ostringstream os;
    tc::write_bench_csv(os, rows);
    if (verified) {
      *verified = 1;
      for (const auto& r : rows) if (!r.verified_ok) *verified = 0;
    }
    const std::string text = os.str();
    if (static_cast<std::int64_t>(text.size()) + 1 > cap) return 4;
    std::memcpy(csv, text.c_str(), text.size() + 1);
    return 0;
  }
  TCF_GUARD(csv, cap)
}

}  // extern "C"
