// L3/L4 on the device: the "b200" KernelBackend and the plan executor.
//
// The reference executor walks the plan's loop nest and issues one CPU BLAS
// call per slice (src/executor.cpp:287-369, run_range :102-283). Here the
// contraction is lowered once (lower.cpp) and executed as permutations + one
// device launch through the C-ABI (tcb.h). Host C++ only: no CUDA headers.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>

#include "tc/contract.hpp"
#include "staging.hpp"
#include "tcb.h"

namespace tc {
namespace {
// TC_EXEC_TRACE=1 (diagnostics): host timestamps of the phases of a call
// (ms since the call began) on stderr
const bool kExecTrace = std::getenv("TC_EXEC_TRACE") != nullptr;
thread_local std::chrono::steady_clock::time_point g_exec_t0 = std::chrono::steady_clock::now();
// TC_STREAM_TIMELINE=1 (diagnostics): device timestamps of the streamed
// paths' copies and contractions (timed events), printed when the call waits
struct Timeline {
  const bool on = std::getenv("TC_STREAM_TIMELINE") != nullptr;
  std::vector<std::pair<std::string, void*>> marks;
  void mark(const std::string& what, void* stream) {
    if (!on) return;
    void* e = nullptr;
    if (tcb_event_create_timed(&e) != TCB_OK) return;
    tcb_event_record(e, stream);
    marks.emplace_back(what, e);
  }
  void print() {
    if (!on || marks.empty()) return;
    for (auto& m : marks) {
      float ms = 0.f;
      tcb_event_elapsed(marks.front().second, m.second, &ms);
      std::fprintf(stderr, "timeline %-28s %9.3f ms\n", m.first.c_str(), ms);
    }
    for (auto& m : marks) tcb_event_destroy(m.second);
    marks.clear();
  }
};
void exec_mark(const char* what) {
  if (kExecTrace)
    std::fprintf(stderr, "execute %-22s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                           g_exec_t0).count());
}

// Map a C-ABI status to the reference's exception types.
void check(int status, const char* what) {
  if (status == TCB_OK) return;
  std::string msg = tcb_last_error();
  if (msg.empty()) msg = what;
  if (status == TCB_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(std::string(what) + ": " + msg);
}

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(std::int64_t bytes) { check(tcb_alloc(&p, bytes), "device allocation"); }
  ~DevBuf() { tcb_free(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  double* d() const { return static_cast<double*>(p); }
};

class B200Backend final : public KernelBackend {
 public:
  explicit B200Backend(const B200Options& o) : opt_(o) {}
  const std::string& name() const override {
    static const std::string n = "b200";
    return n;
  }
  const B200Options& options() const { return opt_; }

  // Fault injection (B200Options::fail_after_launches).
  void tick(const char* where) const {
    if (opt_.fail_after_launches < 0) return;
    std::lock_guard<std::mutex> g(mu_);
    if (ops_++ >= opt_.fail_after_launches)
      throw std::runtime_error(std::string("synthetic device fault in ") + where);
  }

  void gemm(bool ta, bool tb, std::int64_t m, std::int64_t n, std::int64_t k, double alpha,
            const double* a, std::int64_t lda, const double* b, std::int64_t ldb, double beta,
            double* c, std::int64_t ldc) const override {
    check(tcb_init(opt_.device), "tcb_init");
    // validate with the device layer's reference-compatible checks first
    const std::int64_t a_rows = ta ? k : m, a_cols = ta ? m : k;
    const std::int64_t b_rows = tb ? n : k, b_cols = tb ? k : n;
    if (m < 0 || n < 0 || k < 0) throw std::invalid_argument("gemm: negative dimension");
    if (lda < std::max<std::int64_t>(1, a_rows)) throw std::invalid_argument("gemm: lda below row count");
    if (ldb < std::max<std::int64_t>(1, b_rows)) throw std::invalid_argument("gemm: ldb below row count");
    if (ldc < std::max<std::int64_t>(1, m)) throw std::invalid_argument("gemm: ldc below row count");
    tick("gemm");
    if (m == 0 || n == 0) return;
    const std::int64_t na = a_cols > 0 ? lda * (a_cols - 1) + a_rows : 0;
    const std::int64_t nb = b_cols > 0 ? ldb * (b_cols - 1) + b_rows : 0;
    const std::int64_t nc = ldc * (n - 1) + m;
    DevBuf da(std::max<std::int64_t>(na, 1) * 8), db(std::max<std::int64_t>(nb, 1) * 8),
        dc(nc * 8);
    if (na) check(tcb_h2d(da.p, a, na * 8), "gemm upload");
    if (nb) check(tcb_h2d(db.p, b, nb * 8), "gemm upload");
    check(tcb_h2d(dc.p, c, nc * 8), "gemm upload");
    check(tcb_dgemm(ta, tb, m, n, k, alpha, da.d(), lda, db.d(), ldb, beta, dc.d(), ldc), "gemm");
    check(tcb_d2h(c, dc.p, nc * 8), "gemm download");
  }

  void gemv(bool trans, std::int64_t m, std::int64_t n, double alpha, const double* a,
            std::int64_t lda, const double* x, std::int64_t incx, double beta, double* y,
            std::int64_t incy) const override {
    check(tcb_init(opt_.device), "tcb_init");
    if (m < 0 || n < 0) throw std::invalid_argument("gemv: negative dimension");
    if (lda < std::max<std::int64_t>(1, m)) throw std::invalid_argument("gemv: lda below row count");
    tick("gemv");
    const std::int64_t ylen = trans ? n : m, xlen = trans ? m : n;
    if (ylen == 0) return;
    const std::int64_t na = n > 0 ? lda * (n - 1) + m : 0;
    const std::int64_t nx = xlen > 0 ? (xlen - 1) * std::abs(incx) + 1 : 0;
    const std::int64_t ny = (ylen - 1) * std::abs(incy) + 1;
    DevBuf da(std::max<std::int64_t>(na, 1) * 8), dx(std::max<std::int64_t>(nx, 1) * 8),
        dy(ny * 8);
    if (na) check(tcb_h2d(da.p, a, na * 8), "gemv upload");
    if (nx) check(tcb_h2d(dx.p, x, nx * 8), "gemv upload");
    check(tcb_h2d(dy.p, y, ny * 8), "gemv upload");
    check(tcb_dgemv(trans, m, n, alpha, da.d(), lda, dx.d(), incx, beta, dy.d(), incy), "gemv");
    check(tcb_d2h(y, dy.p, ny * 8), "gemv download");
  }

  void ger(std::int64_t m, std::int64_t n, double alpha, const double* x, std::int64_t incx,
           const double* y, std::int64_t incy, double* a, std::int64_t lda) const override {
    check(tcb_init(opt_.device), "tcb_init");
    if (m < 0 || n < 0) throw std::invalid_argument("ger: negative dimension");
    if (lda < std::max<std::int64_t>(1, m)) throw std::invalid_argument("ger: lda below row count");
    tick("ger");
    if (m == 0 || n == 0 || alpha == 0.0) return;
    const std::int64_t nx = (m - 1) * std::abs(incx) + 1, ny = (n - 1) * std::abs(incy) + 1;
    const std::int64_t na = lda * (n - 1) + m;
    DevBuf dx(nx * 8), dy(ny * 8), da(na * 8);
    check(tcb_h2d(dx.p, x, nx * 8), "ger upload");
    check(tcb_h2d(dy.p, y, ny * 8), "ger upload");
    check(tcb_h2d(da.p, a, na * 8), "ger upload");
    check(tcb_dger(m, n, alpha, dx.d(), incx, dy.d(), incy, da.d(), lda), "ger");
    check(tcb_d2h(a, da.p, na * 8), "ger download");
  }

  double dot(std::int64_t k, const double* x, std::int64_t incx, const double* y,
             std::int64_t incy) const override {
    check(tcb_init(opt_.device), "tcb_init");
    tick("dot");
    if (k <= 0) return 0.0;
    const std::int64_t nx = (k - 1) * std::abs(incx) + 1, ny = (k - 1) * std::abs(incy) + 1;
    DevBuf dx(nx * 8), dy(ny * 8);
    check(tcb_h2d(dx.p, x, nx * 8), "dot upload");
    check(tcb_h2d(dy.p, y, ny * 8), "dot upload");
    double r = 0.0;
    check(tcb_ddot(k, dx.d(), incx, dy.d(), incy, &r), "dot");
    return r;
  }

 private:
  B200Options opt_;
  mutable std::mutex mu_;
  mutable int ops_ = 0;
};

}  // namespace

std::unique_ptr<KernelBackend> make_b200_backend(const B200Options& options) {
  return std::make_unique<B200Backend>(options);
}

namespace {
// The B200 backend's BLAS calls behind a type execute() does not lower:
// plans run slice by slice, one device call per slice (execute_sliced).
class SlicedB200 final : public KernelBackend {
 public:
  SlicedB200() : dev_(B200Options{}) {}
  const std::string& name() const override {
    static const std::string n = "b200-sliced";
    return n;
  }
  void gemm(bool ta, bool tb, std::int64_t m, std::int64_t n, std::int64_t k, double alpha,
            const double* a, std::int64_t lda, const double* b, std::int64_t ldb, double beta,
            double* c, std::int64_t ldc) const override {
    dev_.gemm(ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc);
  }
  void gemv(bool trans, std::int64_t m, std::int64_t n, double alpha, const double* a,
            std::int64_t lda, const double* x, std::int64_t incx, double beta, double* y,
            std::int64_t incy) const override {
    dev_.gemv(trans, m, n, alpha, a, lda, x, incx, beta, y, incy);
  }
  void ger(std::int64_t m, std::int64_t n, double alpha, const double* x, std::int64_t incx,
           const double* y, std::int64_t incy, double* a, std::int64_t lda) const override {
    dev_.ger(m, n, alpha, x, incx, y, incy, a, lda);
  }
  double dot(std::int64_t k, const double* x, std::int64_t incx, const double* y,
             std::int64_t incy) const override {
    return dev_.dot(k, x, incx, y, incy);
  }

 private:
  B200Backend dev_;
};
}  // namespace

std::unique_ptr<KernelBackend> make_reference_backend() {
  throw std::invalid_argument(
      "make_reference_backend: the reference's CPU backend is not part of this engine, which "
      "runs on the B200: use make_b200_backend()");
}

std::unique_ptr<KernelBackend> make_eigen_backend() {
  throw std::invalid_argument(
      "make_eigen_backend: the Eigen CPU backend is not part of this engine, which runs on the "
      "B200: use make_b200_backend()");
}

std::unique_ptr<KernelBackend> make_backend(const std::string& name) {
  if (name == "b200" || name == "device") return make_b200_backend();
  if (name == "b200-sliced") return std::make_unique<SlicedB200>();
  if (name == "reference" || name == "external")
    throw std::invalid_argument("backend '" + name +
                                "' is a CPU backend of the reference engine; this engine runs on "
                                "the B200: use make_backend(\"b200\")");
  throw std::invalid_argument("unknown backend '" + name + "'");
}

// --------------------------------------------------------- PreparedContraction

namespace {

tcb_gemm_desc desc_of(const DeviceRecipe& r) {
  tcb_gemm_desc d;
  std::memset(&d, 0, sizeof d);
  d.m = r.m;
  d.n = r.n;
  d.k = r.k;
  d.a_sm = r.a_sm;
  d.a_sk = r.a_sk;
  d.b_sk = r.b_sk;
  d.b_sn = r.b_sn;
  d.c_nrow = static_cast<int32_t>(r.row_ext.size());
  d.c_ncol = static_cast<int32_t>(r.col_ext.size());
  for (std::size_t i = 0; i < r.row_ext.size(); ++i) {
    d.c_row_ext[i] = r.row_ext[i];
    d.c_row_str[i] = r.row_str[i];
  }
  for (std::size_t i = 0; i < r.col_ext.size(); ++i) {
    d.c_col_ext[i] = r.col_ext[i];
    d.c_col_str[i] = r.col_str[i];
  }
  d.nbatch = static_cast<int32_t>(r.bat_ext.size());
  for (std::size_t i = 0; i < r.bat_ext.size(); ++i) {
    d.bat_ext[i] = r.bat_ext[i];
    d.bat_sa[i] = r.bat_sa[i];
    d.bat_sb[i] = r.bat_sb[i];
    d.bat_sc[i] = r.bat_sc[i];
  }
  d.alpha = 1.0;
  d.beta = 0.0;
  if (r.layout == "L4") {
    d.g_m = static_cast<int32_t>(r.gm_ext.size());
    d.g_n = static_cast<int32_t>(r.gn_ext.size());
    d.g_k = static_cast<int32_t>(r.gk_ext.size());
    for (std::size_t i = 0; i < r.gm_ext.size(); ++i) {
      d.m_ext[i] = r.gm_ext[i];
      d.a_m_str[i] = r.gm_sa[i];
    }
    for (std::size_t i = 0; i < r.gn_ext.size(); ++i) {
      d.n_ext[i] = r.gn_ext[i];
      d.b_n_str[i] = r.gn_sb[i];
    }
    for (std::size_t i = 0; i < r.gk_ext.size(); ++i) {
      d.k_ext[i] = r.gk_ext[i];
      d.a_k_str[i] = r.gk_sa[i];
      d.b_k_str[i] = r.gk_sb[i];
    }
  }
  return d;
}

}  // namespace

namespace {
// L4 recipes the device cannot map (the host rules mirror the device's, so
// this is a safety net) are lowered again without index groups.
DeviceRecipe lower_checked(const ValidatedContraction& v, bool* groups_ok,
                           const ValidatedContraction* layout = nullptr) {
  DeviceRecipe r = lower(v, *groups_ok, layout);
  if (r.layout == "L4") {
    const tcb_gemm_desc d = desc_of(r);
    if (tcb_gemm_check(&d) != TCB_OK) {
      *groups_ok = false;
      r = lower(v, false, layout);
    }
  }
  return r;
}

// A contracted label whose slabs the streamed path can upload with one 2-D
// copy per operand and contract in place: the last mode of its contracted
// run in both operands (so slicing it keeps every flattened index group
// chained), extent >= 2, room for two slabs with copy rows of at least 32 KB
// (narrower 2-D rows slow the DMA below the 1-D rate: cfg1's 4 KB rows lost
// to the output-label mode).
// -1 if none; the widest rows win.
constexpr std::int64_t kMinRow = 32 << 10;
// streamed paths: the operand uploaded whole may be pageable up to this size
constexpr std::int64_t kSmallPageable = 4 << 20;
// output-label mode: streamed operand + output bytes per slab (TC_SLAB_MB overrides)
std::int64_t slab_bytes() {
  static const std::int64_t b = [] {
    const char* e = std::getenv("TC_SLAB_MB");
    return (e ? std::max(1LL, std::atoll(e)) : 16LL) << 20;
  }();
  return b;
}

int k_stream_label(const ValidatedContraction& v, std::int64_t min_row = kMinRow) {
  int best = -1;
  std::int64_t best_rows = 0;
  for (int id : v.contracted) {
    const LabelInfo& li = v.labels[static_cast<std::size_t>(id)];
    if (li.extent < 2) continue;
    bool ok = true;
    std::int64_t row_min = std::numeric_limits<std::int64_t>::max();
    for (int side = 0; side < 2 && ok; ++side) {
      const int mode = side ? li.right_mode : li.left_mode;
      const int rank = side ? v.right_rank() : v.left_rank();
      std::int64_t below = 1;
      for (int m = 0; m < mode; ++m)
        below *= (side ? v.label_at_right_mode(m) : v.label_at_left_mode(m)).extent;
      // the next non-unit mode must not be contracted (end of the run)
      for (int m = mode + 1; m < rank; ++m) {
        const LabelInfo& nx = side ? v.label_at_right_mode(m) : v.label_at_left_mode(m);
        if (nx.extent == 1) continue;
        ok = !nx.contracted;
        break;
      }
      row_min = std::min(row_min, below * 8);
    }
    if (!ok || row_min * li.extent < 2 * min_row) continue;
    if (best < 0 || row_min > best_rows) {
      best = id;
      best_rows = row_min;
    }
  }
  return best;
}
}  // namespace


// Streams and events of the streamed path, created once per prepared
// contraction (creating them per call costs more than a small slab).
struct PreparedContraction::Pipes {
  void* up = nullptr;
  void* down = nullptr;
  std::vector<void*> events;
  std::size_t next = 0;
  // per device buffer set (two when successive asynchronous calls alternate
  // between buffer sets): the tail of the last call that used the set — its
  // last contraction and its last download
  void* compute_done[2] = {nullptr, nullptr};
  void* down_done[2] = {nullptr, nullptr};
  bool pending[2] = {false, false};
  // device word the upload stream advances after each slab's copies
  // (tcb_stream_write_value); slab GEMMs wait for it on the device
  // (tcb_gemm_gated), so the compute stream holds only GEMMs and consecutive
  // slab GEMMs overlap under programmatic dependent launch
  std::uint64_t* gate = nullptr;
  std::uint64_t gate_epoch = 0;
  bool gate_ok = true;
  Pipes() {
    check(tcb_stream_create(&up), "stream");
    check(tcb_stream_create(&down), "stream");
    void* g = nullptr;
    if (tcb_alloc(&g, 8) == TCB_OK && tcb_memset0(g, 8) == TCB_OK && tcb_sync() == TCB_OK)
      gate = static_cast<std::uint64_t*>(g);
    else
      gate_ok = false;
    for (int i = 0; i < 2; ++i) {
      check(tcb_event_create(&compute_done[i]), "event");
      check(tcb_event_create(&down_done[i]), "event");
    }
  }
  ~Pipes() {
    if (down) tcb_stream_sync(down);
    if (up) tcb_stream_sync(up);
    tcb_free(gate);
    for (void* e : events) tcb_event_destroy(e);
    for (int i = 0; i < 2; ++i) {
      if (compute_done[i]) tcb_event_destroy(compute_done[i]);
      if (down_done[i]) tcb_event_destroy(down_done[i]);
    }
    tcb_stream_destroy(up);
    tcb_stream_destroy(down);
  }
  // order this call after the pending one that used buffer set `set`:
  // uploads after its contractions (they overwrite operands those read),
  // contractions after its downloads (they overwrite the output those read).
  // With one set that is the previous call, whose download drain then overlaps
  // this call's first uploads; with two sets it is the call before that, so
  // this call's uploads overlap the previous call's contractions as well.
  void follow(void* compute, int set) {
    if (!pending[set]) return;
    check(tcb_stream_wait_event(up, compute_done[set]), "event");
    check(tcb_stream_wait_event(compute, down_done[set]), "event");
  }
  // end of a call: wait for it, or leave it pending
  void finish(void* compute, bool wait, int set) {
    check(tcb_event_record(compute_done[set], compute), "event");
    check(tcb_event_record(down_done[set], down), "event");
    if (wait) {
      check(tcb_stream_sync(down), "sync");
      pending[0] = pending[1] = false;
    } else {
      pending[set] = true;
    }
  }
  void drain() {
    if (pending[0] || pending[1]) check(tcb_stream_sync(down), "sync");
    pending[0] = pending[1] = false;
  }
  void* event() {
    if (next == events.size()) {
      void* e = nullptr;
      check(tcb_event_create(&e), "event");
      events.push_back(e);
    }
    return events[next++];
  }
};

namespace {
constexpr int kPipesPoolDevices = 64;
constexpr std::size_t kPipesPoolPerDevice = 8;
std::mutex g_pipes_mu;
// leaked on purpose: pooled streams live as long as the process (no
// destruction order against the CUDA runtime at exit)
std::vector<void*>* const g_pipes_free = new std::vector<void*>[kPipesPoolDevices];
}  // namespace

std::unique_ptr<PreparedContraction::Pipes> PreparedContraction::acquire_pipes(int device) {
  if (device >= 0 && device < kPipesPoolDevices) {
    std::lock_guard<std::mutex> lock(g_pipes_mu);
    auto& v = g_pipes_free[device];
    if (!v.empty()) {
      std::unique_ptr<Pipes> p(static_cast<Pipes*>(v.back()));
      v.pop_back();
      return p;
    }
  }
  return std::make_unique<Pipes>();
}

void PreparedContraction::release_pipes(int device, std::unique_ptr<Pipes> p) {
  if (!p) return;
  // idle before reuse: nothing pending, both copy streams drained
  p->drain();
  if (tcb_stream_sync(p->up) != TCB_OK || tcb_stream_sync(p->down) != TCB_OK) return;  // dropped
  p->next = 0;
  if (device >= 0 && device < kPipesPoolDevices) {
    std::lock_guard<std::mutex> lock(g_pipes_mu);
    auto& v = g_pipes_free[device];
    if (v.size() < kPipesPoolPerDevice) {
      v.push_back(p.release());
      return;
    }
  }
}

PreparedContraction::PreparedContraction(const ValidatedContraction& v, int device)
    : v_(v), device_(device) {
  check(tcb_init(device_), "tcb_init");
  exec_mark("prepare: init");
  recipe_ = lower_checked(v, &groups_ok_);
  exec_mark("prepare: lowered");
  nl_ = 1;
  for (int m = 0; m < v.left_rank(); ++m) nl_ *= v.label_at_left_mode(m).extent;
  nr_ = 1;
  for (int m = 0; m < v.right_rank(); ++m) nr_ *= v.label_at_right_mode(m).extent;
  no_ = 1;
  for (std::int64_t e : v.output_extents()) no_ *= e;
  if (recipe_.row_ext.size() > TCB_MAX_DIMS || recipe_.col_ext.size() > TCB_MAX_DIMS ||
      recipe_.bat_ext.size() > TCB_MAX_DIMS)
    throw std::invalid_argument("contraction needs more than 6 index groups per role");
  void* p = nullptr;
  try {
    check(tcb_alloc(&p, nl_ * 8), "device allocation");
    dl_ = static_cast<double*>(p);
    exec_mark("prepare: alloc left");
    check(tcb_alloc(&p, nr_ * 8), "device allocation");
    dr_ = static_cast<double*>(p);
    exec_mark("prepare: alloc right");
    check(tcb_alloc(&p, no_ * 8), "device allocation");
    do_ = static_cast<double*>(p);
    exec_mark("prepare: alloc out");
    for (const PermuteStep& ps : recipe_.permutes) {
      check(tcb_alloc(&p, ps.elements * 8), "device allocation");
      (ps.right ? pr_ : pl_) = static_cast<double*>(p);
    }
  } catch (...) {
    tcb_free(dl_);
    tcb_free(dr_);
    tcb_free(do_);
    tcb_free(pl_);
    tcb_free(pr_);
    throw;
  }
}

PreparedContraction::~PreparedContraction() {
  tcb_init(device_);
  tcb_sync();
  try {
    release_pipes(device_, std::move(pipes_));
  } catch (...) {  // drain() reports a failed sync by throwing: drop the pipes
  }
  tcb_free(dl_);
  tcb_free(dr_);
  tcb_free(do_);
  tcb_free(pl_);
  tcb_free(pr_);
  tcb_free(dl2_);
  tcb_free(dr2_);
  tcb_free(do2_);
  tcb_free(pl2_);
  tcb_free(pr2_);
}

// Successive asynchronous streamed calls alternate between two device buffer
// sets (allocated on the first such call, skipped when they do not fit), so a
// call's uploads and contractions never wait for the previous call's
// contractions and downloads — only for those of the call before it.
void PreparedContraction::flip_buffers() {
  if (dbuf_ < 0) {
    dbuf_ = 0;
    auto grab = [](std::int64_t n) {
      void* p = nullptr;
      if (n > 0 && tcb_alloc(&p, n * 8) != TCB_OK) throw std::bad_alloc();
      return static_cast<double*>(p);
    };
    try {
      dl2_ = grab(nl_);
      dr2_ = grab(nr_);
      do2_ = grab(no_);
      for (const PermuteStep& ps : recipe_.permutes) (ps.right ? pr2_ : pl2_) = grab(ps.elements);
      dbuf_ = 1;
    } catch (const std::bad_alloc&) {
      for (double** q : {&dl2_, &dr2_, &do2_, &pl2_, &pr2_}) {
        tcb_free(*q);
        *q = nullptr;
      }
    }
  }
  if (dbuf_ != 1) return;
  std::swap(dl_, dl2_);
  std::swap(dr_, dr2_);
  std::swap(do_, do2_);
  std::swap(pl_, pl2_);
  std::swap(pr_, pr2_);
  set_ ^= 1;
}

std::int64_t PreparedContraction::permuted_bytes() const {
  std::int64_t b = 0;
  for (const PermuteStep& ps : recipe_.permutes) b += ps.elements * 8;
  return b;
}

void PreparedContraction::upload(const double* left, const double* right) {
  check(tcb_init(device_), "tcb_init");
  if (pipes_) pipes_->drain();
  host_to_device(dl_, left, nl_ * 8, nullptr);
  host_to_device(dr_, right, nr_ * 8, nullptr);
}

void PreparedContraction::run() {
  check(tcb_init(device_), "tcb_init");
  if (pipes_) pipes_->drain();
  const std::int64_t before = tcb_launch_count();
  run_permutes();
  run_contraction();
  launches_ = tcb_launch_count() - before;
}

void PreparedContraction::run_permutes() {
  check(tcb_init(device_), "tcb_init");
  for (const PermuteStep& ps : recipe_.permutes)
    check(tcb_permute(static_cast<int>(ps.ext.size()), ps.ext.data(), ps.src_str.data(),
                      ps.right ? dr_ : dl_, ps.right ? pr_ : pl_),
          "permute");
}

void PreparedContraction::run_contraction() {
  check(tcb_init(device_), "tcb_init");
  const double* a = pl_ ? pl_ : dl_;
  const double* b = pr_ ? pr_ : dr_;
  const tcb_gemm_desc d = desc_of(recipe_);
  check(tcb_gemm(&d, a, b, do_), "contraction");
}

static tcb_gemm_desc scattered_desc(const DeviceRecipe& r, std::int64_t no, int parts,
                             std::int64_t part_stride) {
  tcb_gemm_desc d = desc_of(r);
  if (parts < 1) throw std::invalid_argument("run_scattered: parts must be >= 1");
  if (parts == 1) return d;
  // The output's outermost label lives at the high end of the output
  // sub-index with the largest stride (column-major storage).
  int which = -1, at = -1;  // 0 rows, 1 columns, 2 batch
  std::int64_t best = -1;
  auto scan = [&](int w, int n, const std::int64_t* ext, const std::int64_t* str) {
    for (int i = 0; i < n; ++i)
      if (ext[i] > 1 && str[i] > best) best = str[i], which = w, at = i;
  };
  scan(0, d.c_nrow, d.c_row_ext, d.c_row_str);
  scan(1, d.c_ncol, d.c_col_ext, d.c_col_str);
  scan(2, d.nbatch, d.bat_ext, d.bat_sc);
  if (which < 0) throw std::invalid_argument("run_scattered: the output has no label to split");
  std::int64_t* ext = which == 0 ? d.c_row_ext : which == 1 ? d.c_col_ext : d.bat_ext;
  std::int64_t* str = which == 0 ? d.c_row_str : which == 1 ? d.c_col_str : d.bat_sc;
  int32_t& cnt = which == 0 ? d.c_nrow : which == 1 ? d.c_ncol : d.nbatch;
  const std::int64_t e = ext[at], s = str[at];
  // the outermost label's extent: the sub-index spans strides s .. no
  if (no % s || (no / s) % e || (e * s) != no)
    throw std::invalid_argument("run_scattered: the output's outermost label is not the top of "
                                "an output sub-index");
  const std::int64_t block = no / parts;
  if (no % parts || block % s)
    throw std::invalid_argument("run_scattered: the outermost output label's extent must divide "
                                "evenly into " + std::to_string(parts) + " blocks");
  if (part_stride < block)
    throw std::invalid_argument("run_scattered: part stride below the block size");
  if (cnt >= TCB_MAX_DIMS)
    throw std::invalid_argument("run_scattered: too many output sub-indices");
  // sub-index (e, s) -> (e/parts, s) then (parts, part_stride)
  for (int i = cnt; i > at + 1; --i) {
    ext[i] = ext[i - 1];
    str[i] = str[i - 1];
    if (which == 2) {
      d.bat_sa[i] = d.bat_sa[i - 1];
      d.bat_sb[i] = d.bat_sb[i - 1];
    }
  }
  ext[at] = e / parts;
  ext[at + 1] = parts;
  str[at + 1] = part_stride;
  if (which == 2) {  // a batch label also addresses the operands
    d.bat_sa[at + 1] = d.bat_sa[at] * (e / parts);
    d.bat_sb[at + 1] = d.bat_sb[at] * (e / parts);
  }
  ++cnt;
  return d;
}

void PreparedContraction::run_scattered(double* base, int parts, std::int64_t part_stride) {
  check(tcb_init(device_), "tcb_init");
  if (pipes_) pipes_->drain();
  const tcb_gemm_desc d = scattered_desc(recipe_, no_, parts, part_stride);
  const std::int64_t before = tcb_launch_count();
  run_permutes();
  check(tcb_gemm(&d, pl_ ? pl_ : dl_, pr_ ? pr_ : dr_, base), "contraction");
  launches_ = tcb_launch_count() - before;
}

void PreparedContraction::download(double* out) {
  check(tcb_init(device_), "tcb_init");
  if (pipes_) pipes_->drain();
  device_to_host(out, do_, no_ * 8, nullptr);
}

void PreparedContraction::sync() {
  check(tcb_init(device_), "tcb_init");
  if (pipes_) pipes_->drain();
  check(tcb_sync(), "sync");
}


int PreparedContraction::run_streamed(const double* left, const double* right, double* out,
                                      int slabs, bool wait) {
  check(tcb_init(device_), "tcb_init");
  if (!wait || dbuf_ == 1) flip_buffers();
  // Two ways to stream (chosen once): slabs of the output's outermost label
  // (below: the other operand is uploaded whole first, output slabs go down
  // as they complete) or slabs of a contracted label (run_streamed_k: both
  // operands stream, C accumulates on the device and goes down at the end).
  // The one that leaves fewer bytes outside the overlap wins.
  if (stream_mode_ == -1) {
    stream_mode_ = 0;
    // unoverlapped bytes of the output-label mode: the operand uploaded whole
    std::int64_t other = nl_ + nr_;
    int outer = -1;  // the output's outermost label when it is its operand's outermost mode
    const auto& outs = v_.spec.output.indices;
    if (!outs.empty()) {
      const int id = v_.label_index(outs.back().label);
      const LabelInfo& li = v_.labels[static_cast<std::size_t>(id)];
      const bool l = li.left_mode >= 0;
      if ((l ? li.left_mode == v_.left_rank() - 1 : li.right_mode == v_.right_rank() - 1) &&
          li.extent >= 2) {
        other = l ? nr_ : nl_;
        outer = id;
      }
    }
    // a free label elsewhere in the tensors whose slabs go up / down by 2-D
    // copies may leave a smaller operand outside the overlap (cfg4: slabs of
    // b stream A and C, only B goes up whole — instead of A for the output's
    // outermost label j)
    int fs = 0;
    const int fl = recipe_.permutes.empty() ? pick_free_label(&fs) : -1;
    if (fl >= 0 && fl != outer) {
      const LabelInfo& li = v_.labels[static_cast<std::size_t>(fl)];
      const std::int64_t o = li.left_mode >= 0 ? nr_ : nl_;
      if (o < other) {
        other = o;
        stream_mode_ = -2 - fl;
        f_slabs_ = fs;
      }
    }
    // (copy rows of 4 KB still move at the PCIe rate in large copies,
    // tools/pcie.py; where the contraction outweighs the uploads that is
    // enough — a plain product with K < 8192 has no 32 KB rows to offer;
    // 6144^3: 19.8 -> 17.6 ms. At 0.8 x the uploads 4096^3 lost 13 %: 1.1 x)
    const double t_gpu0 = static_cast<double>(flop_count(v_)) / 3.4e13;
    const double t_up0 = static_cast<double>(nl_ + nr_) * 8.0 / 5.5e10;
    static const bool narrow = getenv("TC_STREAM_K_NO_NARROW") == nullptr;  // diagnostics
    const std::int64_t min_row = (narrow && t_gpu0 >= 1.1 * t_up0) ? (4 << 10) : kMinRow;
    const int kl = recipe_.permutes.empty() ? k_stream_label(v_, min_row) : -1;
    // contracted-label slabs when the output is no larger than the operand the
    // other modes upload whole (equal sizes — square matrix products — included:
    // 12288^3 130.9 -> 122.1 ms, 16384^3 285.7 -> 278.5; with a larger output
    // its download outlasts the last slab's contraction: 16384^2 x 8192 144 vs
    // 160 ms, tools/gpu/run85.sh)
    // ... or, with a larger output, when the contraction is long enough that a
    // merged last slab (at most half of the label, run_streamed_k) hides the
    // result's download: download time <= 0.4 x contraction time
    // (TC_STREAM_K_DOWN=<fraction>, diagnostics)
    static const double k_down =
        getenv("TC_STREAM_K_DOWN") ? atof(getenv("TC_STREAM_K_DOWN")) : 0.4;
    const double t_gpu = static_cast<double>(flop_count(v_)) / 3.4e13;
    const double t_down = static_cast<double>(no_) * 8.0 / 5.5e10;
    // (an output exactly as large as that operand — square products — only
    // when the contraction outweighs the uploads: a transfer-bound square
    // product would wait for C's download after the last slab;
    // TC_STREAM_K_SQUARE=always|never overrides, diagnostics)
    const double t_up = static_cast<double>(nl_ + nr_) * 8.0 / 5.5e10;
    static const char* sq = getenv("TC_STREAM_K_SQUARE");
    const bool square_ok = sq ? sq[0] == 'a' : t_gpu >= 1.1 * t_up;
    if (kl >= 0 && (no_ < other || (no_ == other && square_ok) || t_down <= k_down * t_gpu))
      stream_mode_ = 1 + kl;
  }
  if (stream_mode_ > 0) return run_streamed_k(left, right, out, slabs, stream_mode_ - 1, wait);
  if (stream_mode_ <= -2)
    return run_streamed_f(left, right, out, slabs > 0 ? slabs : -f_slabs_, -2 - stream_mode_,
                          wait);  // a negative count: chosen here, not by the caller
  // the stream label: outermost output label, outermost mode of its operand
  const auto& outs = v_.spec.output.indices;
  int label = outs.empty() ? -1 : v_.label_index(outs.back().label);
  bool on_left = false;
  if (label >= 0) {
    const LabelInfo& li = v_.labels[static_cast<std::size_t>(label)];
    on_left = li.left_mode >= 0;
    const int rank = on_left ? v_.left_rank() : v_.right_rank();
    const int mode = on_left ? li.left_mode : li.right_mode;
    if (mode != rank - 1 || li.extent < 2) label = -1;
  }
  if (label >= 0) {
    // a permuted streamed operand must keep the label outermost (contiguous slabs)
    const std::int64_t E = v_.labels[static_cast<std::size_t>(label)].extent;
    for (const PermuteStep& ps : recipe_.permutes)
      if (ps.right != on_left &&
          !(ps.ext.back() == E && ps.src_str.back() * E == (on_left ? nl_ : nr_)))
        label = -1;
  }
  const bool auto_slabs = slabs <= 0;
  if (label >= 0 && slabs <= 0) {
    // auto (decided once per prepared contraction): ~16 MB per slab in the
    // busier copy direction, up to 64 slabs, but no thinner than keeps both slab
    // sizes' GEMM tiles (128x128) as full as the whole contraction's — cfg4's
    // 64 one-j slabs would leave every tile half empty
    if (auto_slabs_ < 0) {
      // the busier copy direction sets the slab size (16 MB of it per slab)
      const std::int64_t bytes = std::max(on_left ? nl_ : nr_, no_) * 8;
      int want = static_cast<int>(std::min<std::int64_t>(64, bytes / slab_bytes()));
      // two slabs from 8 MB on: the second slab's upload overlaps the first
      // slab's contraction (cfg1: 16.8 MB of B)
      if (want < 2 && bytes >= (8LL << 20)) want = 2;
      const std::int64_t E = v_.labels[static_cast<std::size_t>(label)].extent;
      auto tile_eff = [&](std::int64_t e) {
        ValidatedContraction sv = v_;
        sv.labels[static_cast<std::size_t>(label)].extent = e;
        bool ok = groups_ok_;
        const DeviceRecipe r = lower_checked(sv, &ok);
        if (r.m == 1 || r.n == 1) return 1.0;  // GEMV / DOT: no tiles
        const double pm = static_cast<double>((r.m + 127) / 128 * 128);
        const double pn = static_cast<double>((r.n + 127) / 128 * 128);
        return static_cast<double>(r.m) * static_cast<double>(r.n) / (pm * pn);
      };
      const double full = tile_eff(E);
      want = static_cast<int>(std::min<std::int64_t>(want, E));
      for (; want >= 2; --want) {
        const std::int64_t lo = E / want, hi = (E + want - 1) / want;
        if (tile_eff(lo) >= 0.95 * full && (hi == lo || tile_eff(hi) >= 0.95 * full)) break;
      }
      auto_slabs_ = want;
    }
    slabs = auto_slabs_;
  }
  int pinned_l = 0, pinned_r = 0, pinned_o = 0;
  tcb_host_is_pinned(left, &pinned_l);
  tcb_host_is_pinned(right, &pinned_r);
  tcb_host_is_pinned(out, &pinned_o);
  // the streamed operand and the output must be page-locked; the operand that
  // goes up whole first may be pageable when small (tc::execute's operands:
  // only large tensor blocks are pinned)
  const bool other_ok = (on_left ? pinned_r : pinned_l) ||
                        (on_left ? nr_ : nl_) * 8 <= kSmallPageable;
  if (label < 0 || slabs < 2 || !((on_left ? pinned_l : pinned_r) && pinned_o && other_ok)) {
    upload(left, right);
    run();
    download(out);
    return 1;
  }
  const std::int64_t E = v_.labels[static_cast<std::size_t>(label)].extent;
  slabs = static_cast<int>(std::min<std::int64_t>(slabs, E));
  // per-unit-of-label element counts (the label is outermost, so slabs are
  // contiguous in the streamed operand and in the output)
  const std::int64_t s_elems = (on_left ? nl_ : nr_) / E;
  const std::int64_t o_elems = no_ / E;

  // sub-contraction recipes for the two slab sizes
  auto sub_recipe = [&](std::int64_t e) {
    ValidatedContraction sv = v_;
    sv.labels[static_cast<std::size_t>(label)].extent = e;
    bool ok = groups_ok_;
    return lower_checked(sv, &ok);
  };
  // Slab extents: equal slabs; when the slab count was chosen here and the
  // contraction outweighs the copies (a large plain matrix product), a
  // doubling ramp of small first slabs and its mirror at the end, as in
  // run_streamed_f (transfer-bound contractions gain nothing from it: cfg2,
  // cfg3 measured, profiles/r02_experiments.jsonl).
  std::vector<std::int64_t> sched;
  for (int i = 0; i < slabs; ++i) sched.push_back(E / slabs + (i < E % slabs ? 1 : 0));
  {
    static const bool no_ramp = getenv("TC_NO_SLAB_RAMP") != nullptr;
    static const std::int64_t ramp_div =
        getenv("TC_SLAB_RAMP_DIV") ? std::max(2, atoi(getenv("TC_SLAB_RAMP_DIV"))) : 4;
    const std::int64_t nominal = (E + slabs - 1) / slabs;
    const double t_gpu = static_cast<double>(flop_count(v_)) / 3.4e13;
    const double t_copy =
        static_cast<double>(std::max(on_left ? nl_ : nr_, no_)) * 8.0 / 5.5e10;
    std::vector<std::int64_t> ramp;
    for (std::int64_t e = std::max<std::int64_t>(1, nominal / ramp_div); e < nominal; e *= 2)
      ramp.push_back(e);
    std::int64_t ramp_sum = 0;
    for (std::int64_t e : ramp) ramp_sum += e;
    if (auto_slabs && !no_ramp && !ramp.empty() && t_gpu >= 0.8 * t_copy &&
        E >= 2 * ramp_sum + 2 * nominal) {
      sched = ramp;
      std::int64_t rest = E - 2 * ramp_sum;
      while (rest > 0) {
        std::int64_t e = std::min(rest, nominal);
        if (rest - e > 0 && rest - e < (nominal + 1) / 2) e = rest;  // no sliver
        sched.push_back(e);
        rest -= e;
      }
      for (auto it = ramp.rbegin(); it != ramp.rend(); ++it) sched.push_back(*it);
    }
  }
  // slab recipes (one per distinct extent) must permute exactly the operands
  // the full recipe does (its permutation buffers are the ones allocated)
  auto same_permutes = [&](const DeviceRecipe& x) {
    if (x.permutes.size() != recipe_.permutes.size()) return false;
    for (std::size_t i = 0; i < x.permutes.size(); ++i)
      if (x.permutes[i].right != recipe_.permutes[i].right) return false;
    return true;
  };
  std::map<std::int64_t, DeviceRecipe> slab_recipes;
  bool recipes_ok = true;
  for (std::int64_t e : sched)
    if (!slab_recipes.count(e)) {
      auto it = slab_recipes.emplace(e, sub_recipe(e)).first;
      recipes_ok = recipes_ok && same_permutes(it->second);
    }
  if (!recipes_ok) {
    upload(left, right);
    run();
    download(out);
    return 1;
  }
  slabs = static_cast<int>(sched.size());

  exec_mark("o-slabs: lowered");
  if (!pipes_) pipes_ = acquire_pipes(device_);
  Pipes& h = *pipes_;
  exec_mark("o-slabs: pipes");
  h.next = 0;
  void* compute = tcb_current_stream();
  void* up = h.up;
  void* down = h.down;
  h.follow(compute, set_);
  const std::int64_t before = tcb_launch_count();
  // the other operand: whole, first; its permutation (if any) once
  const double* other_host = on_left ? right : left;
  double* other_dev = on_left ? dr_ : dl_;
  check(tcb_memcpy_async(other_dev, other_host, (on_left ? nr_ : nl_) * 8, up), "upload");
  double* stream_dev = on_left ? dl_ : dr_;
  const double* stream_host = on_left ? left : right;
  bool other_permuted = false;
  std::int64_t e0 = 0;
  for (int s = 0; s < slabs; ++s) {
    const std::int64_t e = sched[static_cast<std::size_t>(s)];
    const DeviceRecipe& r = slab_recipes.at(e);
    check(tcb_memcpy_async(stream_dev + e0 * s_elems, stream_host + e0 * s_elems,
                           e * s_elems * 8, up),
          "upload");
    void* ready = h.event();
    check(tcb_event_record(ready, up), "event");
    check(tcb_stream_wait_event(compute, ready), "event");
    // permutations: the other operand's once, the streamed operand's per slab
    const double* a = dl_;
    const double* b = dr_;
    for (const PermuteStep& ps : r.permutes) {
      const bool streamed = ps.right != on_left;
      double* dst = ps.right ? pr_ : pl_;
      if (streamed) {
        const std::int64_t off = e0 * (ps.elements / e);
        check(tcb_permute(static_cast<int>(ps.ext.size()), ps.ext.data(), ps.src_str.data(),
                          stream_dev + e0 * s_elems, dst + off),
              "permute");
      } else if (!other_permuted) {
        const PermuteStep& full = [&]() -> const PermuteStep& {
          for (const PermuteStep& q : recipe_.permutes)
            if (q.right == ps.right) return q;
          return ps;
        }();
        check(tcb_permute(static_cast<int>(full.ext.size()), full.ext.data(),
                          full.src_str.data(), other_dev, dst),
              "permute");
        other_permuted = true;
      }
      (ps.right ? b : a) = dst;
    }
    // the streamed operand (permuted or not) and C at this slab's offset
    const std::int64_t s_off = [&]() {
      for (const PermuteStep& ps : r.permutes)
        if (ps.right != on_left) return e0 * (ps.elements / e);
      return e0 * s_elems;
    }();
    if (on_left) a += s_off;
    else b += s_off;
    tcb_gemm_desc d = desc_of(r);
    check(tcb_gemm(&d, a, b, do_ + e0 * o_elems), "contraction");
    void* done = h.event();
    check(tcb_event_record(done, compute), "event");
    check(tcb_stream_wait_event(down, done), "event");
    check(tcb_memcpy_async(out + e0 * o_elems, do_ + e0 * o_elems, e * o_elems * 8, down),
          "download");
    e0 += e;
  }
  exec_mark("o-slabs: enqueued");
  h.finish(compute, wait, set_);
  exec_mark("o-slabs: finished");
  launches_ = tcb_launch_count() - before;
  return slabs;
}

// Geometry of `label` in a column-major tensor: (elements below its mode,
// elements above it); (0, 0) when the tensor does not carry it. which: 0 left,
// 1 right, 2 output.
static std::pair<std::int64_t, std::int64_t> label_geom(const ValidatedContraction& v,
                                                       int label, int which) {
  std::vector<std::int64_t> ext;
  int mode = -1;
  if (which == 2) {
    const auto& outs = v.spec.output.indices;
    for (std::size_t m = 0; m < outs.size(); ++m) {
      const int id = v.label_index(outs[m].label);
      ext.push_back(v.labels[static_cast<std::size_t>(id)].extent);
      if (id == label) mode = static_cast<int>(m);
    }
  } else {
    const LabelInfo& li = v.labels[static_cast<std::size_t>(label)];
    mode = which ? li.right_mode : li.left_mode;
    const int rank = which ? v.right_rank() : v.left_rank();
    for (int m = 0; m < rank; ++m)
      ext.push_back((which ? v.label_at_right_mode(m) : v.label_at_left_mode(m)).extent);
  }
  if (mode < 0) return {0, 0};
  std::int64_t below = 1, above = 1;
  for (int m = 0; m < static_cast<int>(ext.size()); ++m) {
    if (m < mode) below *= ext[static_cast<std::size_t>(m)];
    if (m > mode) above *= ext[static_cast<std::size_t>(m)];
  }
  return {below, above};
}

// The free label run_streamed_f streams (and its slab count), -1 if none: the
// one whose other operand (uploaded whole before the pipeline starts) is
// smallest, among labels whose slabs (a) move as 2-D copies of rows of at
// least 32 KB in the operand carrying them and in the output, (b) keep the
// GEMM tiles of both slab sizes >= 95 % as full as the whole contraction's,
// (c) lower to the same recipe kind without permutations.
int PreparedContraction::pick_free_label(int* slabs_out) const {
  int best = -1, best_slabs = 0;
  std::int64_t best_other = 0;
  const auto& outs = v_.spec.output.indices;
  for (const auto& ix : outs) {
    const int id = v_.label_index(ix.label);
    const LabelInfo& li = v_.labels[static_cast<std::size_t>(id)];
    const std::int64_t E = li.extent;
    if (E < 2) continue;
    const bool on_left = li.left_mode >= 0;
    const auto [bx, ax] = label_geom(v_, id, on_left ? 0 : 1);
    const auto [bc, ac] = label_geom(v_, id, 2);
    const std::int64_t nx = on_left ? nl_ : nr_, other = on_left ? nr_ : nl_;
    if (best >= 0 && other >= best_other) continue;
    int want = static_cast<int>(std::clamp<std::int64_t>(std::max(nx, no_) * 8 / slab_bytes(),
                                                         2, 64));
    want = static_cast<int>(std::min<std::int64_t>(want, E));
    if (ax > 1) want = static_cast<int>(std::min<std::int64_t>(want, bx * 8 * E / kMinRow));
    if (ac > 1) want = static_cast<int>(std::min<std::int64_t>(want, bc * 8 * E / kMinRow));
    auto slab_ok = [&](std::int64_t e, double full) {
      ValidatedContraction sv = v_;
      sv.labels[static_cast<std::size_t>(id)].extent = e;
      bool ok = groups_ok_;
      const DeviceRecipe r = lower_checked(sv, &ok, &v_);
      if (!r.permutes.empty() || r.layout != recipe_.layout) return false;
      if (r.m == 1 || r.n == 1) return true;
      const double pm = static_cast<double>((r.m + 127) / 128 * 128);
      const double pn = static_cast<double>((r.n + 127) / 128 * 128);
      return static_cast<double>(r.m) * static_cast<double>(r.n) / (pm * pn) >= 0.95 * full;
    };
    double full = 1.0;
    if (recipe_.m > 1 && recipe_.n > 1)
      full = static_cast<double>(recipe_.m) * static_cast<double>(recipe_.n) /
             (static_cast<double>((recipe_.m + 127) / 128 * 128) *
              static_cast<double>((recipe_.n + 127) / 128 * 128));
    for (; want >= 2; --want) {
      const std::int64_t lo = E / want, hi = (E + want - 1) / want;
      if (slab_ok(lo, full) && (hi == lo || slab_ok(hi, full))) break;
    }
    if (want < 2) continue;
    best = id;
    best_other = other;
    best_slabs = want;
  }
  *slabs_out = best_slabs;
  return best;
}

// Streamed evaluation over slabs of free label `label`: the operand not
// carrying it goes up whole first; slab s of the operand carrying it goes up
// (one 2-D copy: `above` rows of below*e elements at pitch below*E) while slab
// s-1 is contracted in place (the slab recipe lowered with the whole tensors'
// strides) and slab s-2 of the output comes down the same way.
int PreparedContraction::run_streamed_f(const double* left, const double* right, double* out,
                                        int slabs, int label, bool wait) {
  const LabelInfo& li = v_.labels[static_cast<std::size_t>(label)];
  const std::int64_t E = li.extent;
  const bool on_left = li.left_mode >= 0;
  const bool auto_slabs = slabs < 0;
  slabs = static_cast<int>(std::clamp<std::int64_t>(slabs < 0 ? -slabs : slabs, 1, E));
  int pinned_l = 0, pinned_r = 0, pinned_o = 0;
  tcb_host_is_pinned(left, &pinned_l);
  tcb_host_is_pinned(right, &pinned_r);
  tcb_host_is_pinned(out, &pinned_o);
  const bool other_ok = (on_left ? pinned_r : pinned_l) ||
                        (on_left ? nr_ : nl_) * 8 <= kSmallPageable;
  if (slabs < 2 || !((on_left ? pinned_l : pinned_r) && pinned_o && other_ok)) {
    upload(left, right);
    run();
    download(out);
    return 1;
  }
  const auto [bx, ax] = label_geom(v_, label, on_left ? 0 : 1);
  const auto [bc, ac] = label_geom(v_, label, 2);
  std::map<std::int64_t, DeviceRecipe> recipes;  // one per distinct slab extent
  std::vector<std::int64_t> sizes;
  for (int i = 0; i < slabs; ++i) sizes.push_back(E / slabs + (i < E % slabs ? 1 : 0));
  // When the contraction, not the copies, bounds the call (cfg4: 61 ms of DMMA
  // over 39 ms of PCIe each way), what stays outside the overlap is the first
  // slab's upload and the last slab's download — a slab each (134 MB, 2.4 ms).
  // A doubling ramp of small first slabs and its mirror at the end shrink both
  // to a quarter (slab counts chosen here only; starting at an eighth measured 1 ms slower on cfg4: TC_SLAB_RAMP_DIV; rows of the 2-D copies stay
  // >= 4 KB, which move at the full PCIe rate). TC_NO_SLAB_RAMP=1: equal slabs.
  static const bool no_ramp = getenv("TC_NO_SLAB_RAMP") != nullptr;
  if (auto_slabs && !no_ramp) {
    const std::int64_t nominal = (E + slabs - 1) / slabs;
    const double t_gpu = static_cast<double>(flop_count(v_)) / 3.4e13;
    const double t_copy = static_cast<double>(std::max(on_left ? nl_ : nr_, no_)) * 8.0 / 5.5e10;
    const std::int64_t min_e = std::max<std::int64_t>(
        1, (4096 + 8 * std::min(bx, bc) - 1) / (8 * std::min(bx, bc)));
    std::vector<std::int64_t> ramp;
    static const std::int64_t ramp_div =
        getenv("TC_SLAB_RAMP_DIV") ? std::max(2, atoi(getenv("TC_SLAB_RAMP_DIV"))) : 4;
    for (std::int64_t e = std::max(min_e, nominal / ramp_div); e < nominal; e *= 2)
      ramp.push_back(e);
    std::int64_t ramp_sum = 0;
    for (std::int64_t e : ramp) ramp_sum += e;
    if (!ramp.empty() && t_gpu >= 0.8 * t_copy && E >= 2 * ramp_sum + 2 * nominal) {
      sizes = ramp;
      std::int64_t rest = E - 2 * ramp_sum;
      while (rest > 0) {
        std::int64_t e = std::min(rest, nominal);
        if (rest - e > 0 && rest - e < (nominal + 1) / 2) e = rest;  // no sliver
        sizes.push_back(e);
        rest -= e;
      }
      for (auto it = ramp.rbegin(); it != ramp.rend(); ++it) sizes.push_back(*it);
      slabs = static_cast<int>(sizes.size());
    }
  }
  for (const std::int64_t e : sizes) {
    if (recipes.count(e)) continue;
    ValidatedContraction sv = v_;
    sv.labels[static_cast<std::size_t>(label)].extent = e;
    bool ok = groups_ok_;
    DeviceRecipe r = lower_checked(sv, &ok, &v_);
    if (!r.permutes.empty()) {  // not expected (checked when the label was picked)
      upload(left, right);
      run();
      download(out);
      return 1;
    }
    recipes.emplace(e, std::move(r));
  }
  if (!pipes_) pipes_ = acquire_pipes(device_);
  Pipes& h = *pipes_;
  h.next = 0;
  void* compute = tcb_current_stream();
  h.follow(compute, set_);
  const std::int64_t before = tcb_launch_count();
  double* x_dev = on_left ? dl_ : dr_;
  const double* x_host = on_left ? left : right;
  check(tcb_memcpy_async(on_left ? dr_ : dl_, on_left ? right : left, (on_left ? nr_ : nl_) * 8,
                         h.up),
        "upload");
  std::int64_t e0 = 0;
  for (int s = 0; s < slabs; ++s) {
    const std::int64_t e = sizes[static_cast<std::size_t>(s)];
    check(tcb_memcpy2d_async(x_dev + e0 * bx, bx * E * 8, x_host + e0 * bx, bx * E * 8,
                             bx * e * 8, ax, h.up),
          "upload");
    void* ready = h.event();
    check(tcb_event_record(ready, h.up), "event");
    check(tcb_stream_wait_event(compute, ready), "event");
    const tcb_gemm_desc d = desc_of(recipes.at(e));
    const double* a = on_left ? dl_ + e0 * bx : dl_;
    const double* b = on_left ? dr_ : dr_ + e0 * bx;
    check(tcb_gemm(&d, a, b, do_ + e0 * bc), "contraction");
    void* done = h.event();
    check(tcb_event_record(done, compute), "event");
    check(tcb_stream_wait_event(h.down, done), "event");
    check(tcb_memcpy2d_async(out + e0 * bc, bc * E * 8, do_ + e0 * bc, bc * E * 8, bc * e * 8,
                             ac, h.down),
          "download");
    e0 += e;
  }
  exec_mark("f-slabs: enqueued");
  h.finish(compute, wait, set_);
  exec_mark("f-slabs: finished");
  launches_ = tcb_launch_count() - before;
  return slabs;
}

// Streamed evaluation over slabs of contracted label `label`: slab s of each
// operand (one 2-D copy: rows of stride*e elements at pitch stride*E) goes up
// on the copy stream while slab s-1 is contracted; the slab GEMMs accumulate
// into C on the device (beta = 1 after the first) and C goes down once.
int PreparedContraction::run_streamed_k(const double* left, const double* right, double* out,
                                        int slabs, int label, bool wait) {
  const LabelInfo& kl = v_.labels[static_cast<std::size_t>(label)];
  const std::int64_t E = kl.extent;
  const bool auto_slabs = slabs <= 0;
  if (auto_slabs)  // ~4 MB of operand data per slab, 2..64 slabs
    slabs = static_cast<int>(std::clamp<std::int64_t>((nl_ + nr_) * 8 / (4LL << 20), 2, 64));
  slabs = static_cast<int>(std::min<std::int64_t>(slabs, E));
  int pinned_l = 0, pinned_r = 0, pinned_o = 0;
  tcb_host_is_pinned(left, &pinned_l);
  tcb_host_is_pinned(right, &pinned_r);
  tcb_host_is_pinned(out, &pinned_o);
  // (stride of the label, rows above it) per operand, in elements
  auto geom = [&](bool right_side) {
    const int mode = right_side ? kl.right_mode : kl.left_mode;
    const int rank = right_side ? v_.right_rank() : v_.left_rank();
    std::int64_t below = 1, above = 1;
    for (int m = 0; m < rank; ++m) {
      const std::int64_t e = (right_side ? v_.label_at_right_mode(m) : v_.label_at_left_mode(m)).extent;
      if (m < mode) below *= e;
      if (m > mode) above *= e;
    }
    return std::make_pair(below, above);
  };
  const auto [sa, ha] = geom(false);
  const auto [sb, hb] = geom(true);
  // copy rows of at least 32 KB per slab (4 KB when the engine chose the
  // slabs for a contraction that outweighs its uploads, as in run_streamed)
  {
    const double t_gpu0 = static_cast<double>(flop_count(v_)) / 3.4e13;
    const double t_up0 = static_cast<double>(nl_ + nr_) * 8.0 / 5.5e10;
    static const bool narrow = getenv("TC_STREAM_K_NO_NARROW") == nullptr;
    const std::int64_t min_row =
        (auto_slabs && narrow && t_gpu0 >= 1.1 * t_up0) ? (4 << 10) : kMinRow;
    slabs = static_cast<int>(std::min<std::int64_t>(slabs, std::min(sa, sb) * 8 * E / min_row));
  }
  if (slabs < 2 || !(pinned_l && pinned_r && pinned_o)) {
    upload(left, right);
    run();
    download(out);
    return 1;
  }
  // Slab extents: a short ramp (1, 2, 4, ... up to the nominal extent) so the
  // first contraction starts after a small upload instead of a whole nominal
  // slab's, then nominal slabs (a tail below half the nominal merges into the
  // slab before it).
  // An explicit slab count gets equal slabs. Slab offsets stay multiples of 2
  // when a row is an odd number of doubles (16-byte aligned bases: the tensor
  // maps of in-place index groups need them).
  std::vector<std::int64_t> sizes;
  if (!auto_slabs) {
    for (int i = 0; i < slabs; ++i) sizes.push_back(E / slabs + (i < E % slabs ? 1 : 0));
  } else {
    // Nominal slabs are an eighth of the label: long slab GEMMs run at the
    // whole contraction's efficiency (cfg5: 2048 k-blocks per tile, the
    // stream-K tail applies; 64 slabs of 256 k-blocks lost 3 % to per-slab
    // wave tails and epilogues). The ramp grows by 1.5x per slab so each
    // upload (PCIe, ~55 GB/s) stays shorter than the previous slab's
    // contraction.
    const std::int64_t unit = ((sa | sb) & 1) ? 2 : 1;
    const std::int64_t nominal = std::max<std::int64_t>(unit, (E + 7) / 8 / unit * unit);
    // the ramp opens with a slab of at least 256 contracted elements (16
    // k-blocks per tile): below that a slab GEMM is all epilogue (a plain
    // 8192^3 product ramping from 2 spent 3 ms in ten slabs that rewrite the
    // whole 537 MB of C for k = 2..94 each); cfg5's label unit is already 512
    const std::int64_t per_unit = std::max<std::int64_t>(1, recipe_.k / E);
    const std::int64_t row_e = (4096 + 8 * std::min(sa, sb) - 1) / (8 * std::min(sa, sb));
    const std::int64_t open_e = std::min(
        nominal,
        (std::max((256 + per_unit - 1) / per_unit, row_e) + unit - 1) / unit * unit);
    std::int64_t rest = E, ramp = std::max(unit, open_e);
    while (rest > 0) {
      std::int64_t e = std::min({rest, ramp / unit * unit, nominal});
      e = std::max(e, std::min(rest, unit));
      if (rest - e > 0 && rest - e < (nominal + 1) / 2) e = rest;
      sizes.push_back(e);
      rest -= e;
      ramp = std::max(ramp + unit, ramp * 3 / 2);
    }
    // The last slab's contraction hides the result's download (its column
    // blocks go down as they finish, below) only if it lasts as long as that
    // download: where the contraction outweighs the copies, trailing slabs
    // merge until it does (8192^3: C takes 9.8 ms to download, an eighth of
    // the contraction 4 ms; cfg5: 122 ms against 9.8, nothing to merge).
    static const bool no_merge = getenv("TC_NO_LAST_MERGE") != nullptr;  // diagnostics
    const double t_gpu = static_cast<double>(flop_count(v_)) / 3.4e13;
    const double t_up = static_cast<double>(nl_ + nr_) * 8.0 / 5.5e10;
    const double t_down = static_cast<double>(no_) * 8.0 / 5.5e10;
    if (!no_merge && t_gpu >= 0.8 * t_up)
      while (sizes.size() > 2 &&
             t_gpu * static_cast<double>(sizes.back()) / static_cast<double>(E) < t_down &&
             2 * (sizes.back() + sizes[sizes.size() - 2]) <= E) {
        sizes[sizes.size() - 2] += sizes.back();
        sizes.pop_back();
      }
    slabs = static_cast<int>(sizes.size());
  }
  // The last slab's contraction is split into column blocks of the output's
  // outermost label, each downloaded as soon as it is final, so the result's
  // download overlaps the last contractions instead of following them.
  const auto& outs = v_.spec.output.indices;
  const int o_label = outs.empty() ? -1 : v_.label_index(outs.back().label);
  const std::int64_t o_ext = o_label < 0 ? 1 : v_.labels[static_cast<std::size_t>(o_label)].extent;
  int parts = auto_slabs ? static_cast<int>(std::min<std::int64_t>(8, o_ext)) : 1;
  std::map<std::pair<std::int64_t, std::int64_t>, DeviceRecipe> recipes;  // (slab, block) extents
  auto recipe = [&](std::int64_t e, std::int64_t ob) -> const DeviceRecipe* {
    const auto key = std::make_pair(e, ob);
    if (auto it = recipes.find(key); it != recipes.end()) return &it->second;
    ValidatedContraction sv = v_;
    sv.labels[static_cast<std::size_t>(label)].extent = e;
    if (ob > 0) sv.labels[static_cast<std::size_t>(o_label)].extent = ob;
    bool ok = groups_ok_;
    DeviceRecipe r = lower_checked(sv, &ok, &v_);
    if (!r.permutes.empty()) return nullptr;  // not expected (the full recipe permutes nothing)
    return &recipes.emplace(key, std::move(r)).first->second;
  };
  exec_mark("k-slabs: sized");
  bool lowered = true;
  for (std::int64_t e : sizes) lowered = lowered && recipe(e, 0) != nullptr;
  for (int q = 0; q < parts && parts >= 2; ++q)
    lowered = lowered && recipe(sizes.back(), o_ext * (q + 1) / parts - o_ext * q / parts);
  if (!lowered) {
    upload(left, right);
    run();
    download(out);
    return 1;
  }
  // element strides of the output's outermost label in A, B and C
  std::int64_t o_sa = 0, o_sb = 0, o_sc = 1;
  if (parts >= 2) {
    const LabelInfo& li = v_.labels[static_cast<std::size_t>(o_label)];
    auto stride_in = [&](bool right_side, int mode) {
      std::int64_t st = 1;
      for (int m = 0; m < mode; ++m)
        st *= (right_side ? v_.label_at_right_mode(m) : v_.label_at_left_mode(m)).extent;
      return st;
    };
    if (li.left_mode >= 0) o_sa = stride_in(false, li.left_mode);
    if (li.right_mode >= 0) o_sb = stride_in(true, li.right_mode);
    o_sc = no_ / o_ext;
    if ((o_sa | o_sb | o_sc) & 1) parts = 1;  // block offsets would break 16-byte alignment
  }
  exec_mark("k-slabs: lowered");
  if (!pipes_) pipes_ = acquire_pipes(device_);
  Pipes& h = *pipes_;
  exec_mark("k-slabs: pipes");
  h.next = 0;
  void* compute = tcb_current_stream();
  h.follow(compute, set_);
  const std::int64_t before = tcb_launch_count();
  Timeline tl;
  tl.mark("start", h.up);
  std::int64_t e0 = 0;
  for (int s = 0; s < slabs; ++s) {
    const std::int64_t e = sizes[static_cast<std::size_t>(s)];
    check(tcb_memcpy2d_async(dl_ + e0 * sa, sa * E * 8, left + e0 * sa, sa * E * 8, sa * e * 8,
                             ha, h.up),
          "upload");
    check(tcb_memcpy2d_async(dr_ + e0 * sb, sb * E * 8, right + e0 * sb, sb * E * 8, sb * e * 8,
                             hb, h.up),
          "upload");
    tl.mark("slab " + std::to_string(s) + " (" + std::to_string(e) + ") up", h.up);
    // the slab's contraction waits for its uploads: on the device through the
    // gate where available, else through an event on the compute stream
    bool gated = h.gate_ok && tcb_stream_write_value(h.up, h.gate, h.gate_epoch + 1) == TCB_OK;
    if (gated) {
      ++h.gate_epoch;
    } else {
      h.gate_ok = false;
      void* ready = h.event();
      check(tcb_event_record(ready, h.up), "event");
      check(tcb_stream_wait_event(compute, ready), "event");
    }
    auto gemm = [&](const tcb_gemm_desc& d, const double* a, const double* b, double* c) {
      check(gated ? tcb_gemm_gated(&d, a, b, c, h.gate, h.gate_epoch) : tcb_gemm(&d, a, b, c),
            "contraction");
    };
    const double beta = s == 0 ? 0.0 : 1.0;
    if (s + 1 < slabs || parts < 2) {
      tcb_gemm_desc d = desc_of(*recipe(e, 0));
      d.beta = beta;
      gemm(d, dl_ + e0 * sa, dr_ + e0 * sb, do_);
      tl.mark("slab " + std::to_string(s) + " gemm", compute);
    } else {
      for (int q = 0; q < parts; ++q) {
        const std::int64_t b0 = o_ext * q / parts, b1 = o_ext * (q + 1) / parts;
        tcb_gemm_desc d = desc_of(*recipe(e, b1 - b0));
        d.beta = beta;
        gemm(d, dl_ + e0 * sa + b0 * o_sa, dr_ + e0 * sb + b0 * o_sb, do_ + b0 * o_sc);
        void* block_done = h.event();
        check(tcb_event_record(block_done, compute), "event");
        check(tcb_stream_wait_event(h.down, block_done), "event");
        tl.mark("part " + std::to_string(q) + " gemm", compute);
        check(tcb_memcpy_async(out + b0 * o_sc, do_ + b0 * o_sc, (b1 - b0) * o_sc * 8, h.down),
              "download");
        tl.mark("part " + std::to_string(q) + " down", h.down);
      }
    }
    e0 += e;
  }
  if (parts < 2) {
    void* done = h.event();
    check(tcb_event_record(done, compute), "event");
    check(tcb_stream_wait_event(h.down, done), "event");
    check(tcb_memcpy_async(out, do_, no_ * 8, h.down), "download");
  }
  exec_mark("k-slabs: enqueued");
  h.finish(compute, wait, set_);
  exec_mark("k-slabs: finished");
  if (wait) tl.print();
  launches_ = tcb_launch_count() - before;
  return slabs;
}

// ------------------------------------------------------------------ execute

namespace {

// plan / contraction consistency (reference: src/executor.cpp:292-297); the
// operand extents are checked by the Tensor overload
void check_plan(const ExecutionPlan& plan, const ValidatedContraction& v) {
  if (plan.label_extents.size() != v.labels.size())
    throw std::invalid_argument("plan does not match contraction");
  for (std::size_t i = 0; i < v.labels.size(); ++i)
    if (v.labels[i].extent != plan.label_extents[i])
      throw std::invalid_argument("extent drift between planning and execution on label '" +
                                  v.labels[i].label + "'");
}

// One contraction on the device over host storage: lowered once, then either
// the streamed pipeline (H2D / DMMA / D2H overlapped; needs page-locked
// storage) or upload + run + download.
void run_on_device(const B200Backend& dev, const ValidatedContraction& v, const double* left,
                   const double* right, double* out, bool streamed, ExecutionStats& st,
                   const std::chrono::steady_clock::time_point& t0) {
  g_exec_t0 = t0;
  auto mark = [](const char* what) { exec_mark(what); };
  try {
    dev.tick("execute");
    PreparedContraction pc(v, dev.options().device);
    mark("prepare");
    if (streamed) {
      pc.run_streamed(left, right, out);
      mark("streamed");
    } else {
      pc.upload(left, right);
      mark("upload");
      pc.run();
      mark("run");
      pc.download(out);
      mark("download");
    }
    st.kernel_calls = pc.launches_last_run();
    st.packed_bytes = pc.permuted_bytes();
  } catch (const std::invalid_argument&) {
    throw;
  } catch (const std::exception& e) {
    throw std::runtime_error(std::string(e.what()) + " while executing " +
                             lower(v).summary() + " for " + unparse(v.spec));
  }
}

bool host_pinned(const void* p) {
  int pinned = 0;
  return p && tcb_host_is_pinned(p, &pinned) == TCB_OK && pinned;
}

}  // namespace

ExecutionStats execute_into(const ExecutionPlan& plan, const ValidatedContraction& v,
                            const double* left, const double* right, double* out,
                            const KernelBackend& backend, int workers) {
  check_plan(plan, v);
  const auto t0 = std::chrono::steady_clock::now();
  ExecutionStats st;
  st.flops = plan.flops;
  if (const auto* dev = dynamic_cast<const B200Backend*>(&backend)) {
    // caller-owned storage is never registered here: it streams when the
    // caller page-locked it (tcb_host_register / tcb_host_alloc)
    static const bool off = std::getenv("TC_NO_PIN") != nullptr;
    const bool streamed =
        !off && host_pinned(out) && (host_pinned(left) || host_pinned(right));
    run_on_device(*dev, v, left, right, out, streamed, st, t0);
    exec_mark("released");
  } else {
    std::int64_t n = 1;
    for (std::int64_t e : v.output_extents()) n *= e;
    std::fill(out, out + n, 0.0);
    execute_sliced(plan, v, left, right, out, backend, workers, st);
  }
  st.wall_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return st;
}

std::pair<Tensor, ExecutionStats> execute(const ExecutionPlan& plan,
                                          const ValidatedContraction& v, const Tensor& left,
                                          const Tensor& right, const KernelBackend& backend,
                                          int workers) {
  // plan/operand consistency (reference: src/executor.cpp:292-303)
  check_plan(plan, v);
  for (const LabelInfo& li : v.labels) {
    if (li.left_mode >= 0 && left.extent(li.left_mode) != li.extent)
      throw std::invalid_argument("left operand extent drift on label '" + li.label + "'");
    if (li.right_mode >= 0 && right.extent(li.right_mode) != li.extent)
      throw std::invalid_argument("right operand extent drift on label '" + li.label + "'");
  }
  const auto t0 = std::chrono::steady_clock::now();
  ExecutionStats st;
  st.flops = plan.flops;
  const auto* dev = dynamic_cast<const B200Backend*>(&backend);
  if (!dev) {
    // any other KernelBackend: the reference's loop over kernel calls
    Tensor out(v.output_extents(), v.output_variance(), v.spec.output.name);
    execute_sliced(plan, v, left.data(), right.data(), out.data(), backend, workers, st);
    st.wall_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return {std::move(out), st};
  }
  Tensor out(v.output_extents(), v.output_variance(), v.spec.output.name,
             Tensor::Uninit{});  // overwritten whole by the download
  // large operands and result page-locked (once per storage block): the
  // streamed path overlaps their transfers with the contraction
  const auto bytes = [](const Tensor& t) { return static_cast<std::size_t>(t.size()) * 8; };
  const bool pl = tensor_storage_pin(left.data(), bytes(left));
  const bool pr = tensor_storage_pin(right.data(), bytes(right));
  const bool po = tensor_storage_pin(out.data(), bytes(out));
  // run_streamed checks the rest (a small operand may stay pageable)
  run_on_device(*dev, v, left.data(), right.data(), out.data(), po && (pl || pr), st, t0);
  st.wall_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return {std::move(out), st};
}

std::vector<SlicingRun> execute_all_slicings(const ValidatedContraction& v, const Tensor& left,
                                             const Tensor& right, const KernelBackend& backend,
                                             std::int64_t work_cap) {
  const std::vector<SlicingOption> opts = enumerate_slicings(v);
  const std::int64_t macs = flop_count(v) / 2;
  if (macs * static_cast<std::int64_t>(opts.size()) > work_cap)
    throw resource_limit_error("slicing sweep work exceeds cap");
  std::vector<SlicingRun> runs;
  runs.reserve(opts.size());
  for (const SlicingOption& o : opts) {
    SlicingRun run;
    run.s_left = o.s_left;
    run.s_right = o.s_right;
    run.kernel = o.report.kernel;
    const ExecutionPlan p = plan(v, PlanPolicy::force_slicing(o.s_left, o.s_right));
    auto [res, st] = execute(p, v, left, right, backend);
    run.result_hash = tensor_hash(res);
    run.stats = st;
    run.result = std::move(res);
    runs.push_back(std::move(run));
  }
  return runs;
}

// tc/oracle.hpp (reference include/tc/oracle.hpp:11-25): the brute-force
// contraction evaluated by the device kernel tcb_contract_naive, bit-identical
// to the reference's src/oracle.cpp:32-94 (same order, no FMA).
Tensor contract_naive(const ValidatedContraction& v, const Tensor& left, const Tensor& right,
                      std::int64_t work_cap, OracleStats* stats) {
  std::int64_t work = 1;
  for (const LabelInfo& l : v.labels) work *= l.extent;
  if (work > work_cap)
    throw resource_limit_error("oracle work exceeds cap: " + std::to_string(work) +
                               " multiply-adds");
  Tensor out(v.output_extents(), v.output_variance(), v.spec.output.name);
  std::vector<std::int64_t> fe, fl, fr, fo, ce, cl, cr;
  for (const auto& ix : v.spec.output.indices) {
    const LabelInfo& li = v.labels[static_cast<std::size_t>(v.label_index(ix.label))];
    fe.push_back(li.extent);
    fl.push_back(li.left_mode >= 0 ? stride_of(left, li.left_mode) : 0);
    fr.push_back(li.right_mode >= 0 ? stride_of(right, li.right_mode) : 0);
    fo.push_back(stride_of(out, li.output_mode));
  }
  for (int id : v.contracted) {
    const LabelInfo& li = v.labels[static_cast<std::size_t>(id)];
    ce.push_back(li.extent);
    cl.push_back(stride_of(left, li.left_mode));
    cr.push_back(stride_of(right, li.right_mode));
  }
  DevBuf dl(std::max<std::int64_t>(left.size(), 1) * 8), dr(std::max<std::int64_t>(right.size(), 1) * 8),
      dout(out.size() * 8);
  check(tcb_h2d(dl.p, left.data(), left.size() * 8), "oracle upload");
  check(tcb_h2d(dr.p, right.data(), right.size() * 8), "oracle upload");
  check(tcb_contract_naive(static_cast<int>(fe.size()), fe.data(), fl.data(), fr.data(),
                           fo.data(), static_cast<int>(ce.size()), ce.data(), cl.data(),
                           cr.data(), dl.d(), dr.d(), dout.d()),
        "contract_naive");
  check(tcb_d2h(out.data(), dout.p, out.size() * 8), "oracle download");
  if (stats) stats->multiply_adds = work;
  return out;
}

std::uint64_t tensor_hash(const Tensor& t) {
  // FNV-1a over the little-endian bytes of each element (src/executor.cpp:371-383)
  std::uint64_t h = 0xcbf29ce484222325ull;
  const unsigned char* bytes = reinterpret_cast<const unsigned char*>(t.data());
  const std::size_t n = static_cast<std::size_t>(t.size()) * sizeof(double);
  for (std::size_t i = 0; i < n; ++i) {
    h ^= bytes[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

double max_rel_error(const Tensor& a, const Tensor& b) {
  if (a.size() != b.size()) return std::numeric_limits<double>::infinity();
  double scale = 1.0, worst = 0.0;
  for (std::int64_t i = 0; i < b.size(); ++i) scale = std::max(scale, std::fabs(b.data()[i]));
  for (std::int64_t i = 0; i < a.size(); ++i)
    worst = std::max(worst, std::fabs(a.data()[i] - b.data()[i]));
  return worst / scale;
}

double rel_frobenius_error(const Tensor& a, const Tensor& b) {
  if (a.size() != b.size()) return std::numeric_limits<double>::infinity();
  long double num = 0, den = 0;
  for (std::int64_t i = 0; i < a.size(); ++i) {
    const long double d = static_cast<long double>(a.data()[i]) - b.data()[i];
    num += d * d;
    den += static_cast<long double>(b.data()[i]) * b.data()[i];
  }
  if (den == 0) return num == 0 ? 0.0 : std::numeric_limits<double>::infinity();
  return static_cast<double>(std::sqrt(num / den));
}

}  // namespace tc
