// The loop-over-kernel driver for any KernelBackend other than the B200 one.
//
// The reference's extension point is the KernelBackend interface: execute()
// walks the plan's loop nest and makes one BLAS call per slice
// (src/executor.cpp:102-283, threads over free slices :330-364). Callers that
// plug in their own backend — the reference tests' FailingBackend
// (tests/test_executor.cpp:240-291), an instrumented or host BLAS — keep that
// behaviour here: same call sequence, beta (0 on the first contracted slice,
// 1 after), slice packing (COPY) and output staging, same ExecutionStats and
// the same " at slice coordinates [..]" error suffix. The B200 backend never
// comes here: execute() lowers its plans to device launches (executor.cpp).
#include <algorithm>
#include <exception>
#include <mutex>
#include <sstream>
#include <thread>

#include "tc/contract.hpp"

namespace tc {
namespace {

// One operand (or the output) as seen by the kernel: the storage strides of
// its kept modes (slicing bit 0) in mode order.
struct Kept {
  std::vector<std::int64_t> ext, str;
};

// A loop of the plan's nest with the storage stride of its label in each
// tensor (0 where the label does not occur).
struct Loop {
  std::int64_t extent = 1;
  std::int64_t sl = 0, sr = 0, so = 0;
};

std::vector<std::int64_t> col_major(const std::vector<std::int64_t>& ext) {
  std::vector<std::int64_t> s(ext.size());
  std::int64_t run = 1;
  for (std::size_t i = 0; i < ext.size(); ++i) {
    s[i] = run;
    run *= ext[i];
  }
  return s;
}

Kept kept_of(const std::vector<std::int64_t>& ext, const SlicingVector& s) {
  const std::vector<std::int64_t> str = col_major(ext);
  Kept k;
  for (std::size_t m = 0; m < ext.size(); ++m)
    if (m >= s.size() || !s[m]) {
      k.ext.push_back(ext[m]);
      k.str.push_back(str[m]);
    }
  return k;
}

// Odometer over a set of loops, last loop fastest (the reference's flat
// decode order, src/executor.cpp:73-84): offsets are updated incrementally.
struct Odometer {
  const std::vector<Loop>* loops;
  std::vector<std::int64_t> at;
  std::int64_t ol = 0, or_ = 0, oo = 0;
  explicit Odometer(const std::vector<Loop>& l) : loops(&l), at(l.size(), 0) {}
  void seek(std::int64_t flat) {
    ol = or_ = oo = 0;
    for (std::size_t i = loops->size(); i-- > 0;) {
      const Loop& d = (*loops)[i];
      at[i] = flat % d.extent;
      flat /= d.extent;
      ol += at[i] * d.sl;
      or_ += at[i] * d.sr;
      oo += at[i] * d.so;
    }
  }
  void next() {
    for (std::size_t i = loops->size(); i-- > 0;) {
      const Loop& d = (*loops)[i];
      if (++at[i] < d.extent) {
        ol += d.sl;
        or_ += d.sr;
        oo += d.so;
        return;
      }
      ol -= (d.extent - 1) * d.sl;
      or_ -= (d.extent - 1) * d.sr;
      oo -= (d.extent - 1) * d.so;
      at[i] = 0;
    }
  }
};

struct Driver {
  const ExecutionPlan& plan;
  const ValidatedContraction& v;
  const double* L;
  const double* R;
  double* O;
  const KernelBackend& be;
  Kept lk, rk, ok;
  std::vector<std::int64_t> lstr, rstr;  // full storage strides of the operands
  std::vector<Loop> free_loops, con_loops;
  std::vector<std::string> names;  // loop-nest labels, nest order
  std::vector<bool> is_con;

  Driver(const ExecutionPlan& p, const ValidatedContraction& vc, const double* l,
         const double* r, double* o, const KernelBackend& b)
      : plan(p), v(vc), L(l), R(r), O(o), be(b) {
    std::vector<std::int64_t> le, re;
    for (int m = 0; m < v.left_rank(); ++m) le.push_back(v.label_at_left_mode(m).extent);
    for (int m = 0; m < v.right_rank(); ++m) re.push_back(v.label_at_right_mode(m).extent);
    const std::vector<std::int64_t> oe = v.output_extents();
    lstr = col_major(le);
    rstr = col_major(re);
    const std::vector<std::int64_t> ostr = col_major(oe);
    lk = kept_of(le, plan.s_left);
    rk = kept_of(re, plan.s_right);
    ok = kept_of(oe, plan.s_output);
    for (const LoopLabel& ll : plan.loop_nest) {
      const LabelInfo& li = v.labels[static_cast<std::size_t>(ll.label)];
      Loop d;
      d.extent = li.extent;
      if (li.left_mode >= 0) d.sl = lstr[static_cast<std::size_t>(li.left_mode)];
      if (li.right_mode >= 0) d.sr = rstr[static_cast<std::size_t>(li.right_mode)];
      if (li.output_mode >= 0) d.so = ostr[static_cast<std::size_t>(li.output_mode)];
      (ll.contracted ? con_loops : free_loops).push_back(d);
      names.push_back(li.label);
      is_con.push_back(ll.contracted);
    }
  }

  std::int64_t ext(int label) const { return v.labels[static_cast<std::size_t>(label)].extent; }

  std::string where(const Odometer& f, const Odometer& c) const {
    std::ostringstream os;
    os << " at slice coordinates [";
    std::size_t fi = 0, ci = 0;
    for (std::size_t i = 0; i < names.size(); ++i)
      os << (i ? ", " : "") << names[i] << '=' << (is_con[i] ? c.at[ci++] : f.at[fi++]);
    os << ']';
    return os.str();
  }

  // A 2-D slice of an operand for the kernel: aliased when its first kept
  // mode is unit-stride, otherwise packed column-major into `scratch` (the
  // COPY of COPY+GEMM / COPY+GEMV, src/executor.cpp:41-59).
  const double* matrix(const double* base, const Kept& k, std::vector<double>& scratch,
                       std::int64_t* ld, ExecutionStats& st) const {
    const std::int64_t rows = k.ext[0], cols = k.ext[1];
    if (k.str[0] == 1) {
      *ld = k.str[1];
      return base;
    }
    scratch.resize(static_cast<std::size_t>(rows * cols));
    double* d = scratch.data();
    for (std::int64_t j = 0; j < cols; ++j) {
      const double* src = base + j * k.str[1];
      for (std::int64_t i = 0; i < rows; ++i) d[i + j * rows] = src[i * k.str[0]];
    }
    st.packed_bytes += rows * cols * 8;
    *ld = rows;
    return d;
  }

  void elementwise(const double* lb, const double* rb, double* ob) const {
    // every kept mode of both slices: left kept (contracted ones carry the
    // right stride too), then right kept free ones (src/executor.cpp:228-265)
    std::vector<Loop> dims;
    const std::vector<std::int64_t> ostr = col_major(v.output_extents());
    for (std::size_t i = 0, m = 0; m < static_cast<std::size_t>(v.left_rank()); ++m) {
      if (m < plan.s_left.size() && plan.s_left[m]) continue;
      const LabelInfo& li = v.label_at_left_mode(static_cast<int>(m));
      Loop d;
      d.extent = lk.ext[i];
      d.sl = lk.str[i++];
      if (li.contracted) d.sr = rstr[static_cast<std::size_t>(li.right_mode)];
      if (li.output_mode >= 0) d.so = ostr[static_cast<std::size_t>(li.output_mode)];
      dims.push_back(d);
    }
    for (std::size_t i = 0, m = 0; m < static_cast<std::size_t>(v.right_rank()); ++m) {
      if (m < plan.s_right.size() && plan.s_right[m]) continue;
      const LabelInfo& li = v.label_at_right_mode(static_cast<int>(m));
      const std::size_t at = i++;
      if (li.contracted) continue;
      Loop d;
      d.extent = rk.ext[at];
      d.sr = rk.str[at];
      if (li.output_mode >= 0) d.so = ostr[static_cast<std::size_t>(li.output_mode)];
      dims.push_back(d);
    }
    std::int64_t space = 1;
    for (const Loop& d : dims) space *= d.extent;
    Odometer e(dims);
    for (std::int64_t t = 0; t < space; ++t, e.next()) ob[e.oo] += lb[e.ol] * rb[e.or_];
  }

  void run(std::int64_t flo, std::int64_t fhi, ExecutionStats& st) const {
    const KernelMap& km = plan.kernel_map;
    std::int64_t cspace = 1;
    for (const Loop& d : con_loops) cspace *= d.extent;
    std::vector<double> sa, sb, stage;
    const bool matrix_out = plan.kernel == KernelKind::Gemm ||
                            plan.kernel == KernelKind::CopyGemm || plan.kernel == KernelKind::Ger;
    Odometer f(free_loops), c(con_loops);
    f.seek(flo);
    for (std::int64_t fi = flo; fi < fhi; ++fi, f.next()) {
      double* cptr = nullptr;
      std::int64_t ldc = 0;
      const bool staged = matrix_out && ok.str[0] != 1;
      if (matrix_out) {
        if (!staged) {
          cptr = O + f.oo;
          ldc = ok.str[1];
        } else {
          stage.assign(static_cast<std::size_t>(ok.ext[0] * ok.ext[1]), 0.0);
          cptr = stage.data();
          ldc = ok.ext[0];
        }
      }
      c.seek(0);
      for (std::int64_t ci = 0; ci < cspace; ++ci, c.next()) {
        const double beta = ci == 0 ? 0.0 : 1.0;
        const double* lb = L + f.ol + c.ol;
        const double* rb = R + f.or_ + c.or_;
        try {
          switch (plan.kernel) {
            case KernelKind::Gemm:
            case KernelKind::CopyGemm: {
              std::int64_t lda = 0, ldb = 0;
              const double* a = matrix(km.a_is_left ? lb : rb, km.a_is_left ? lk : rk, sa, &lda,
                                       st);
              const double* b = matrix(km.a_is_left ? rb : lb, km.a_is_left ? rk : lk, sb, &ldb,
                                       st);
              be.gemm(km.trans_a, km.trans_b, ext(km.m_label), ext(km.n_label), ext(km.k_label),
                      1.0, a, lda, b, ldb, beta, cptr, ldc);
              ++st.kernel_calls;
              break;
            }
            case KernelKind::Gemv:
            case KernelKind::CopyGemv: {
              const Kept& mk = km.matrix_is_left ? lk : rk;
              const Kept& vk = km.matrix_is_left ? rk : lk;
              std::int64_t lda = 0;
              const double* a = matrix(km.matrix_is_left ? lb : rb, mk, sa, &lda, st);
              be.gemv(km.trans_a, mk.ext[0], mk.ext[1], 1.0, a, lda,
                      km.matrix_is_left ? rb : lb, vk.str[0], beta, O + f.oo, ok.str[0]);
              ++st.kernel_calls;
              break;
            }
            case KernelKind::Ger: {
              const Kept& xk = km.a_is_left ? lk : rk;
              const Kept& yk = km.a_is_left ? rk : lk;
              be.ger(ext(km.m_label), ext(km.n_label), 1.0, km.a_is_left ? lb : rb, xk.str[0],
                     km.a_is_left ? rb : lb, yk.str[0], cptr, ldc);
              ++st.kernel_calls;
              break;
            }
            case KernelKind::Dot: {
              const LabelInfo& k1 = v.labels[static_cast<std::size_t>(km.k_label)];
              const std::int64_t lx = lstr[static_cast<std::size_t>(k1.left_mode)];
              const std::int64_t ry = rstr[static_cast<std::size_t>(k1.right_mode)];
              double acc = 0.0;
              if (km.k2_label >= 0) {
                const LabelInfo& k2 = v.labels[static_cast<std::size_t>(km.k2_label)];
                const std::int64_t l2 = lstr[static_cast<std::size_t>(k2.left_mode)];
                const std::int64_t r2 = rstr[static_cast<std::size_t>(k2.right_mode)];
                for (std::int64_t q = 0; q < k2.extent; ++q) {
                  acc += be.dot(k1.extent, lb + q * l2, lx, rb + q * r2, ry);
                  ++st.kernel_calls;
                }
              } else {
                acc = be.dot(k1.extent, lb, lx, rb, ry);
                ++st.kernel_calls;
              }
              O[f.oo] += acc;
              break;
            }
            case KernelKind::Elementwise:
              elementwise(lb, rb, O + f.oo);
              ++st.kernel_calls;
              break;
          }
        } catch (const std::exception& e) {
          throw std::runtime_error(std::string(e.what()) + where(f, c));
        }
      }
      if (staged) {
        for (std::int64_t j = 0; j < ok.ext[1]; ++j)
          for (std::int64_t i = 0; i < ok.ext[0]; ++i)
            O[f.oo + i * ok.str[0] + j * ok.str[1]] = stage[static_cast<std::size_t>(i + j * ok.ext[0])];
        st.staged_bytes += ok.ext[0] * ok.ext[1] * 8;
      }
    }
  }
};

}  // namespace

// Declared in executor.cpp's translation unit via contract.hpp's execute();
// `out` must be zero on entry (DOT, GER and ELEMENTWISE accumulate into it).
void execute_sliced(const ExecutionPlan& plan, const ValidatedContraction& v, const double* left,
                    const double* right, double* out, const KernelBackend& backend, int workers,
                    ExecutionStats& stats) {
  const Driver d(plan, v, left, right, out, backend);
  std::int64_t fspace = 1;
  for (const Loop& l : d.free_loops) fspace *= l.extent;
  const int nw = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(workers, fspace)));
  if (nw == 1) {
    d.run(0, fspace, stats);
    return;
  }
  std::vector<ExecutionStats> per(static_cast<std::size_t>(nw));
  std::vector<std::thread> pool;
  std::exception_ptr first;
  std::mutex mu;
  for (int w = 0; w < nw; ++w)
    pool.emplace_back([&, w] {
      try {
        d.run(fspace * w / nw, fspace * (w + 1) / nw, per[static_cast<std::size_t>(w)]);
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!first) first = std::current_exception();
      }
    });
  for (std::thread& t : pool) t.join();
  if (first) std::rethrow_exception(first);
  for (const ExecutionStats& s : per) {
    stats.kernel_calls += s.kernel_calls;
    stats.packed_bytes += s.packed_bytes;
    stats.staged_bytes += s.staged_bytes;
  }
}

}  // namespace tc
