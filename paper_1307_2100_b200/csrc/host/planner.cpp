// L2 — classification, requirement analysis, slicing enumeration and plans
// (reference: src/planner.cpp:1-538). Results must be identical to the
// reference (tests/test_planner_parity.py diffs both over thousands of
// random contractions), so this file restates its rules:
//   classify            planner.cpp:136-144
//   check_requirements  planner.cpp:146-203   (R1/R2/R3 -> kernel, fallback)
//   enumerate_slicings  planner.cpp:240-284   (<= 2 kept labels per side)
//   plan / pick_best    planner.cpp:379-456   (class recipe + tie-breaks)
//   build_plan          planner.cpp:288-377   (loop nest, kernel map, copies)
//   render_plan         planner.cpp:458-494
//   relayout_advice     planner.cpp:496-536
#include <algorithm>
#include <cctype>
#include <sstream>

#include "tc/contract.hpp"

namespace tc {

std::string to_string(ContractionClass c) {
  static const char* names[] = {"1", "2", "3.1", "3.2"};
  const int i = static_cast<int>(c);
  return (i >= 0 && i < 4) ? names[i] : "?";
}

std::string to_string(KernelKind k) {
  static const char* names[] = {"GEMM", "COPY+GEMM", "GEMV", "COPY+GEMV",
                                "GER",  "DOT",       "ELEMENTWISE"};
  const int i = static_cast<int>(k);
  return (i >= 0 && i < 7) ? names[i] : "?";
}

std::optional<KernelKind> kernel_from_string(const std::string& s) {
  std::string up(s);
  for (char& c : up) c = static_cast<char>(std::toupper(static_cast<unsigned char>(c)));
  static const std::pair<const char*, KernelKind> table[] = {
      {"GEMM", KernelKind::Gemm},       {"COPY+GEMM", KernelKind::CopyGemm},
      {"COPYGEMM", KernelKind::CopyGemm}, {"GEMV", KernelKind::Gemv},
      {"COPY+GEMV", KernelKind::CopyGemv}, {"COPYGEMV", KernelKind::CopyGemv},
      {"GER", KernelKind::Ger},         {"DOT", KernelKind::Dot},
      {"ELEMENTWISE", KernelKind::Elementwise}};
  for (const auto& [n, k] : table)
    if (up == n) return k;
  return std::nullopt;
}

std::string to_string(Fallback f) {
  static const char* names[] = {"none", "F1", "F2", "F3"};
  const int i = static_cast<int>(f);
  return (i >= 0 && i < 4) ? names[i] : "?";
}

namespace {

// Canonical column-major strides of every label in every tensor it addresses
// (0 when absent), computed from the bound extents.
struct Geometry {
  std::vector<std::int64_t> ls, rs, os;  // per label
  std::vector<int> left_at, right_at;    // label id at each mode
  std::vector<int> out_at;

  explicit Geometry(const ValidatedContraction& v) {
    const std::size_t n = v.labels.size();
    ls.assign(n, 0);
    rs.assign(n, 0);
    os.assign(n, 0);
    left_at.assign(static_cast<std::size_t>(v.left_rank()), -1);
    right_at.assign(static_cast<std::size_t>(v.right_rank()), -1);
    out_at.assign(static_cast<std::size_t>(v.output_rank()), -1);
    for (std::size_t i = 0; i < n; ++i) {
      const LabelInfo& li = v.labels[i];
      if (li.left_mode >= 0) left_at[static_cast<std::size_t>(li.left_mode)] = static_cast<int>(i);
      if (li.right_mode >= 0)
        right_at[static_cast<std::size_t>(li.right_mode)] = static_cast<int>(i);
      if (li.output_mode >= 0)
        out_at[static_cast<std::size_t>(li.output_mode)] = static_cast<int>(i);
    }
    fill(v, left_at, ls);
    fill(v, right_at, rs);
    fill(v, out_at, os);
  }
  static void fill(const ValidatedContraction& v, const std::vector<int>& at,
                   std::vector<std::int64_t>& str) {
    std::int64_t run = 1;
    for (int id : at) {
      str[static_cast<std::size_t>(id)] = run;
      run *= v.labels[static_cast<std::size_t>(id)].extent;
    }
  }
};

// Which labels a slicing pair keeps, in the orders the reference uses.
struct Kept {
  std::vector<int> left, right;          // kept labels in mode order
  std::vector<int> pairs;                // kept contracted (left-mode order)
  std::vector<int> lfree, rfree;         // kept free labels per side
  std::vector<int> out;                  // kept labels in output order
  bool left_unit = true, right_unit = true, out_unit = true;  // first kept has stride 1
};

bool label_sliced(const ValidatedContraction& v, int id, const SlicingVector& sl,
                  const SlicingVector& sr) {
  const LabelInfo& li = v.labels[static_cast<std::size_t>(id)];
  return li.left_mode >= 0 ? sl[static_cast<std::size_t>(li.left_mode)] != 0
                           : sr[static_cast<std::size_t>(li.right_mode)] != 0;
}

Kept kept_of(const ValidatedContraction& v, const Geometry& g, const SlicingVector& sl,
             const SlicingVector& sr) {
  Kept k;
  for (std::size_t m = 0; m < g.left_at.size(); ++m) {
    if (sl[m]) continue;
    const int id = g.left_at[m];
    if (k.left.empty()) k.left_unit = g.ls[static_cast<std::size_t>(id)] == 1;
    k.left.push_back(id);
    (v.labels[static_cast<std::size_t>(id)].contracted ? k.pairs : k.lfree).push_back(id);
  }
  for (std::size_t m = 0; m < g.right_at.size(); ++m) {
    if (sr[m]) continue;
    const int id = g.right_at[m];
    if (k.right.empty()) k.right_unit = g.rs[static_cast<std::size_t>(id)] == 1;
    k.right.push_back(id);
    if (!v.labels[static_cast<std::size_t>(id)].contracted) k.rfree.push_back(id);
  }
  for (int id : g.out_at) {
    if (label_sliced(v, id, sl, sr)) continue;
    if (k.out.empty()) k.out_unit = g.os[static_cast<std::size_t>(id)] == 1;
    k.out.push_back(id);
  }
  return k;
}

RequirementReport assess(const Kept& k, const SlicingVector& sl, const SlicingVector& sr,
                         int lrank, int rrank) {
  auto ones = [](const SlicingVector& s) {
    return static_cast<int>(std::count_if(s.begin(), s.end(), [](std::uint8_t b) { return b != 0; }));
  };
  RequirementReport rep;
  rep.r1_ok = (lrank == 0 || sl[0] == 0) && (rrank == 0 || sr[0] == 0);
  rep.r2_ok = ones(sl) == lrank - 2 && ones(sr) == rrank - 2;
  rep.r3_ok = k.lfree.size() == 1 && k.rfree.size() == 1 && k.pairs.size() == 1;
  const std::size_t nl = k.left.size(), nr = k.right.size();
  const bool left_matrix = k.lfree.size() == 1 && nl == 2 && k.rfree.empty() && nr == 1;
  const bool right_matrix = k.rfree.size() == 1 && nr == 2 && k.lfree.empty() && nl == 1;
  if (rep.r2_ok && rep.r3_ok)
    rep.kernel = rep.r1_ok ? KernelKind::Gemm : KernelKind::CopyGemm;
  else if (k.pairs.size() == 1 && (left_matrix || right_matrix))
    rep.kernel = (nl == 2 ? k.left_unit : k.right_unit) ? KernelKind::Gemv : KernelKind::CopyGemv;
  else if (!k.pairs.empty() && k.lfree.empty() && k.rfree.empty())
    rep.kernel = KernelKind::Dot;
  else if (k.pairs.empty() && k.lfree.size() == 1 && k.rfree.size() == 1 && nl == 1 && nr == 1)
    rep.kernel = KernelKind::Ger;
  else
    rep.kernel = KernelKind::Elementwise;

  switch (rep.kernel) {
    case KernelKind::Gemm: rep.fallback = Fallback::None; break;
    case KernelKind::CopyGemm: rep.fallback = Fallback::F1; break;
    default:
      rep.fallback = !rep.r2_ok ? Fallback::F2 : (!rep.r3_ok ? Fallback::F3 : Fallback::None);
  }
  return rep;
}

void check_slicing(const ValidatedContraction& v, const SlicingVector& sl,
                   const SlicingVector& sr) {
  if (static_cast<int>(sl.size()) != v.left_rank() || static_cast<int>(sr.size()) != v.right_rank())
    throw std::invalid_argument("slicing vector length does not match rank");
  for (int id : v.contracted) {
    const LabelInfo& li = v.labels[static_cast<std::size_t>(id)];
    if (sl[static_cast<std::size_t>(li.left_mode)] != sr[static_cast<std::size_t>(li.right_mode)])
      throw std::invalid_argument("contracted label '" + li.label + "' sliced in one tensor only");
  }
}

std::int64_t kernel_size(const ValidatedContraction& v, const Kept& k, KernelKind kind) {
  auto e = [&](int id) { return v.labels[static_cast<std::size_t>(id)].extent; };
  auto prod = [&](const std::vector<int>& ids) {
    std::int64_t x = 1;
    for (int id : ids) x *= e(id);
    return x;
  };
  switch (kind) {
    case KernelKind::Gemm:
    case KernelKind::CopyGemm: return e(k.lfree[0]) * e(k.rfree[0]) * e(k.pairs[0]);
    case KernelKind::Gemv:
    case KernelKind::CopyGemv: return e(k.lfree.empty() ? k.rfree[0] : k.lfree[0]) * e(k.pairs[0]);
    case KernelKind::Ger: return e(k.lfree[0]) * e(k.rfree[0]);
    case KernelKind::Dot: return prod(k.pairs);
    case KernelKind::Elementwise: return prod(k.left) * prod(k.rfree);
  }
  return 0;
}

ExecutionPlan make_plan(const ValidatedContraction& v, ContractionClass cls,
                        const SlicingVector& sl, const SlicingVector& sr,
                        const RequirementReport& rep) {
  const Geometry g(v);
  const Kept k = kept_of(v, g, sl, sr);
  ExecutionPlan p;
  p.cls = cls;
  p.s_left = sl;
  p.s_right = sr;
  p.kernel = rep.kernel;
  p.flops = flop_count(v);
  for (const auto& li : v.labels) p.label_extents.push_back(li.extent);
  for (int id : g.out_at) p.s_output.push_back(label_sliced(v, id, sl, sr) ? 1 : 0);

  // loop nest: sliced free labels (label order) outside, sliced contracted inside
  for (std::size_t id = 0; id < v.labels.size(); ++id) {
    const LabelInfo& li = v.labels[id];
    if (!li.contracted && label_sliced(v, static_cast<int>(id), sl, sr))
      p.loop_nest.push_back({static_cast<int>(id), false, li.extent});
  }
  for (int id : v.contracted)
    if (label_sliced(v, id, sl, sr))
      p.loop_nest.push_back({id, true, v.labels[static_cast<std::size_t>(id)].extent});

  KernelMap& km = p.kernel_map;
  const auto first_kept = [&](bool left) { return left ? k.left.front() : k.right.front(); };
  switch (rep.kernel) {
    case KernelKind::Gemm:
    case KernelKind::CopyGemm:
      km.m_label = k.out[0];
      km.n_label = k.out[1];
      km.k_label = k.pairs[0];
      km.a_is_left = v.labels[static_cast<std::size_t>(km.m_label)].left_mode >= 0;
      km.trans_a = first_kept(km.a_is_left) != km.m_label;
      km.trans_b = first_kept(!km.a_is_left) != km.k_label;
      if (!k.left_unit) p.copies.push_back(CopyTarget::Left);
      if (!k.right_unit) p.copies.push_back(CopyTarget::Right);
      if (!k.out_unit) p.copies.push_back(CopyTarget::OutputStage);
      break;
    case KernelKind::Gemv:
    case KernelKind::CopyGemv:
      km.matrix_is_left = k.left.size() == 2;
      km.m_label = km.matrix_is_left ? k.lfree[0] : k.rfree[0];
      km.k_label = k.pairs[0];
      km.trans_a = first_kept(km.matrix_is_left) != km.m_label;
      if (rep.kernel == KernelKind::CopyGemv)
        p.copies.push_back(km.matrix_is_left ? CopyTarget::Left : CopyTarget::Right);
      break;
    case KernelKind::Ger:
      km.m_label = k.out[0];
      km.n_label = k.out[1];
      km.a_is_left = v.labels[static_cast<std::size_t>(km.m_label)].left_mode >= 0;
      if (!k.out_unit) p.copies.push_back(CopyTarget::OutputStage);
      break;
    case KernelKind::Dot:
      km.k_label = k.pairs[0];
      if (k.pairs.size() == 2) {
        km.k2_label = k.pairs[1];
        // run the dot over the pair that is unit-stride in the left slice
        if (g.ls[static_cast<std::size_t>(k.pairs[1])] == 1) std::swap(km.k_label, km.k2_label);
      }
      break;
    case KernelKind::Elementwise: break;
  }
  return p;
}

// First option (in enumeration order) of an allowed kind with the largest
// kernel-dims product, preferring an unstaged output on ties.
const SlicingOption* best_option(const ValidatedContraction& v,
                                 const std::vector<SlicingOption>& opts,
                                 std::initializer_list<KernelKind> kinds, bool one_pair) {
  const Geometry g(v);
  const SlicingOption* best = nullptr;
  for (const SlicingOption& o : opts) {
    if (std::find(kinds.begin(), kinds.end(), o.report.kernel) == kinds.end()) continue;
    if (one_pair && kept_of(v, g, o.s_left, o.s_right).pairs.size() != 1) continue;
    const bool better =
        !best || o.kernel_dims_product > best->kernel_dims_product ||
        (o.kernel_dims_product == best->kernel_dims_product && best->output_staged &&
         !o.output_staged);
    if (better) best = &o;
  }
  return best;
}

std::string slicing_text(const SlicingVector& s) {
  std::string t = "(";
  for (std::size_t i = 0; i < s.size(); ++i) {
    if (i) t += ", ";
    t += s[i] ? '1' : '0';
  }
  return t + ")";
}

}  // namespace

ContractionClass classify(const ValidatedContraction& v) {
  if (v.delta_left == 0 || v.delta_right == 0)
    return (v.delta_left == 0 && v.delta_right == 0) ? ContractionClass::C1 : ContractionClass::C2;
  const LabelInfo& a = v.label_at_left_mode(0);
  const LabelInfo& b = v.label_at_right_mode(0);
  const bool crossed = a.contracted && b.contracted && a.label != b.label;
  return crossed ? ContractionClass::C31 : ContractionClass::C32;
}

RequirementReport check_requirements(const ValidatedContraction& v, const SlicingVector& s_left,
                                     const SlicingVector& s_right) {
  check_slicing(v, s_left, s_right);
  const Geometry g(v);
  return assess(kept_of(v, g, s_left, s_right), s_left, s_right, v.left_rank(), v.right_rank());
}

std::vector<SlicingOption> enumerate_slicings(const ValidatedContraction& v) {
  const Geometry g(v);
  const int np = v.p;
  const int nl = static_cast<int>(v.left_free.size());
  const int nr = static_cast<int>(v.right_free.size());
  std::vector<SlicingOption> out;
  // keep-masks: bit i of `pk` keeps contracted pair i, of `lk`/`rk` the i-th
  // free label of a side; at most two kept labels per residual slice.
  for (unsigned pk = 0; pk < (1u << np); ++pk) {
    const int kp = __builtin_popcount(pk);
    if (kp > 2) continue;
    for (unsigned lk = 0; lk < (1u << nl); ++lk) {
      if (kp + __builtin_popcount(lk) > 2) continue;
      for (unsigned rk = 0; rk < (1u << nr); ++rk) {
        if (kp + __builtin_popcount(rk) > 2) continue;
        SlicingOption o;
        o.s_left.assign(static_cast<std::size_t>(v.left_rank()), 1);
        o.s_right.assign(static_cast<std::size_t>(v.right_rank()), 1);
        for (int i = 0; i < np; ++i)
          if (pk >> i & 1u) {
            const LabelInfo& li = v.labels[static_cast<std::size_t>(v.contracted[i])];
            o.s_left[static_cast<std::size_t>(li.left_mode)] = 0;
            o.s_right[static_cast<std::size_t>(li.right_mode)] = 0;
          }
        for (int i = 0; i < nl; ++i)
          if (lk >> i & 1u)
            o.s_left[static_cast<std::size_t>(v.labels[static_cast<std::size_t>(v.left_free[i])].left_mode)] = 0;
        for (int i = 0; i < nr; ++i)
          if (rk >> i & 1u)
            o.s_right[static_cast<std::size_t>(v.labels[static_cast<std::size_t>(v.right_free[i])].right_mode)] = 0;
        const Kept k = kept_of(v, g, o.s_left, o.s_right);
        o.report = assess(k, o.s_left, o.s_right, v.left_rank(), v.right_rank());
        o.kernel_dims_product = kernel_size(v, k, o.report.kernel);
        o.output_staged = !k.out_unit;
        out.push_back(std::move(o));
      }
    }
  }
  std::sort(out.begin(), out.end(), [](const SlicingOption& a, const SlicingOption& b) {
    return std::tie(a.s_left, a.s_right) < std::tie(b.s_left, b.s_right);
  });
  return out;
}

ExecutionPlan plan(const ValidatedContraction& v, const PlanPolicy& policy) {
  const ContractionClass cls = classify(v);
  if (policy.mode == PlanPolicy::Mode::ForceSlicing) {
    const RequirementReport rep = check_requirements(v, policy.s_left, policy.s_right);
    return make_plan(v, cls, policy.s_left, policy.s_right, rep);
  }
  const std::vector<SlicingOption> opts = enumerate_slicings(v);
  const SlicingOption* best = nullptr;
  if (policy.mode == PlanPolicy::Mode::ForceKernel) {
    best = best_option(v, opts, {policy.kernel}, false);
    if (!best) {
      if (policy.kernel != KernelKind::Gemm)
        throw kernel_unreachable_error("kernel unreachable: no slicing yields " +
                                       to_string(policy.kernel));
      // name the requirement that blocks GEMM for this class
      std::string req = "R1";
      if (cls == ContractionClass::C1 || cls == ContractionClass::C2)
        req = std::min(v.left_rank(), v.right_rank()) < 2 ? "R2" : "R3";
      throw kernel_unreachable_error(KernelKind::Gemm, req);
    }
  } else {
    switch (cls) {
      case ContractionClass::C32: best = best_option(v, opts, {KernelKind::Gemm}, false); break;
      case ContractionClass::C31: best = best_option(v, opts, {KernelKind::CopyGemm}, false); break;
      case ContractionClass::C2:
        best = best_option(v, opts, {KernelKind::Gemv}, false);
        if (!best) best = best_option(v, opts, {KernelKind::CopyGemv}, false);
        break;
      case ContractionClass::C1: best = best_option(v, opts, {KernelKind::Dot}, true); break;
    }
    if (!best)
      throw std::logic_error("no recipe-conformant slicing found for class " + to_string(cls));
  }
  return make_plan(v, cls, best->s_left, best->s_right, best->report);
}

std::string render_plan(const ExecutionPlan& p, const ValidatedContraction& v) {
  auto name = [&](int id) { return v.labels[static_cast<std::size_t>(id)].label; };
  std::ostringstream os;
  os << "class: " << to_string(p.cls) << '\n'
     << "delta: (" << v.delta_left << ", " << v.delta_right << ")\n"
     << "s_left: " << slicing_text(p.s_left) << '\n'
     << "s_right: " << slicing_text(p.s_right) << '\n'
     << "s_output: " << slicing_text(p.s_output) << '\n'
     << "kernel: " << to_string(p.kernel) << '\n'
     << "loop_nest:";
  if (p.loop_nest.empty()) os << " (none)";
  for (const LoopLabel& l : p.loop_nest)
    os << ' ' << name(l.label) << ':' << (l.contracted ? "contracted" : "free");
  os << "\nkernel_map:";
  const KernelMap& km = p.kernel_map;
  const std::pair<const char*, int> roles[] = {
      {" M=", km.m_label}, {" N=", km.n_label}, {" K=", km.k_label}, {" K2=", km.k2_label}};
  for (const auto& [tag, id] : roles)
    if (id >= 0) os << tag << name(id);
  if (p.kernel == KernelKind::Gemm || p.kernel == KernelKind::CopyGemm)
    os << " transA=" << int(km.trans_a) << " transB=" << int(km.trans_b);
  else if (p.kernel == KernelKind::Gemv || p.kernel == KernelKind::CopyGemv)
    os << " trans=" << int(km.trans_a);
  os << "\ncopies: " << p.copies.size() << "\nflops: " << p.flops << '\n';
  return os.str();
}

std::optional<std::string> relayout_advice(const ValidatedContraction& v) {
  if (classify(v) != ContractionClass::C31) return std::nullopt;
  // A label that may be rotated into an operand's stride-1 slot: any non-mode-0
  // label that is free, or is the partner of the other operand's mode-0 label.
  // Ranking: larger extent, then the right operand, then the lower mode.
  struct Choice {
    bool right = false;
    int mode = 0;
    std::int64_t extent = -1;
  };
  std::optional<Choice> best;
  for (bool right : {true, false}) {
    const int rank = right ? v.right_rank() : v.left_rank();
    const std::string& partner = (right ? v.label_at_left_mode(0) : v.label_at_right_mode(0)).label;
    for (int m = 1; m < rank; ++m) {
      const LabelInfo& li = right ? v.label_at_right_mode(m) : v.label_at_left_mode(m);
      if (li.contracted && li.label != partner) continue;
      const Choice c{right, m, li.extent};
      const bool wins = !best || c.extent > best->extent ||
                        (c.extent == best->extent && c.right && !best->right) ||
                        (c.extent == best->extent && c.right == best->right && c.mode < best->mode);
      if (wins) best = c;
    }
  }
  if (!best) return std::nullopt;
  const TensorExpr& t = best->right ? v.spec.right : v.spec.left;
  const auto& lead = t.indices[static_cast<std::size_t>(best->mode)];
  std::string s = "store " + t.name + " as " + t.name + "[" + variance_char(lead.var) + lead.label;
  for (std::size_t m = 0; m < t.indices.size(); ++m) {
    if (static_cast<int>(m) == best->mode) continue;
    s += ',';
    s += variance_char(t.indices[m].var);
    s += t.indices[m].label;
  }
  return s + "] to reach class 3.2 (direct GEMM, no copies)";
}

}  // namespace tc
