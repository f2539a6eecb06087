// Device lowering: a validated contraction -> one DeviceRecipe (optional
// operand permutations + one batched GEMM with composite output addressing).
//
// This pass has no reference counterpart: the reference executes a plan as a
// loop nest of small BLAS calls (src/executor.cpp:102-283). Here the index
// groups are flattened in place wherever the strides chain:
//   M = left free labels, N = right free labels, K = contracted labels.
//   K must be one contiguous run of modes, in the same label order, in both
//   operands; M must be a run in the left operand, N in the right one.
//   * L1 — every group is a run: one GEMM reads the operands in place
//     (BASELINE cfg1, cfg4, cfg5);
//   * L2 — a free label outside its side's run becomes a batch dimension with
//     per-operand strides (0 where absent): one strided-batched launch (cfg2);
//   * L3 — K is not a run (or the K orders disagree): the offending operand(s)
//     are permuted on the device into [M|N, K] or [K, M|N] order, keeping each
//     operand's unit-stride label innermost so the permutation copies
//     contiguous runs (cfg3: A[a,k,c,l] -> A'[a,c,l,k], B[l,b,k,d] -> B'[l,k,b,d]).
//   * L4 — instead of L3 where the GEMM's tensor maps can describe the groups
//     directly: M = all left free labels, N = all right free labels, K = all
//     contracted labels, each a composite of operand dimensions whose inner
//     sub-index tiles the kernel's TMA boxes (cfg3 reads A[a,k,c,l] and
//     B[l,b,k,d] in place: M=(a,c), N=(b,d), K=(l,k)). No permutation pass.
// The output is never permuted: the GEMM epilogue addresses C through the
// composite row (M labels) and column (N labels) strides. Extent-1 labels are
// dropped first (any coordinate of them is 0).
#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <sstream>

#include "tc/contract.hpp"
#include "tcb.h"

namespace tc {
namespace {

struct Side {
  std::vector<int> modes;              // non-unit label ids in mode order
  std::vector<std::int64_t> stride;    // per label id (canonical), 0 if absent
  std::vector<std::int64_t> extent;    // per label id: iteration extent
  std::int64_t elements = 1;
};

// Strides come from `layout` (the storage the operand lives in: the full
// contraction when v is a slab of it), iteration extents from v.
Side side_of(const ValidatedContraction& v, const ValidatedContraction& layout, bool right) {
  Side s;
  s.stride.assign(v.labels.size(), 0);
  s.extent.assign(v.labels.size(), 1);
  const int rank = right ? v.right_rank() : v.left_rank();
  std::int64_t run = 1, elems = 1;
  for (int m = 0; m < rank; ++m) {
    const LabelInfo& li = right ? v.label_at_right_mode(m) : v.label_at_left_mode(m);
    const LabelInfo& lo = right ? layout.label_at_right_mode(m) : layout.label_at_left_mode(m);
    const int id = v.label_index(li.label);
    s.stride[static_cast<std::size_t>(id)] = run;
    s.extent[static_cast<std::size_t>(id)] = li.extent;
    run *= lo.extent;
    elems *= li.extent;
    if (li.extent > 1) s.modes.push_back(id);
  }
  s.elements = elems;
  return s;
}

// Maximal runs of consecutive (non-unit) modes whose labels satisfy `in` and
// whose strides chain (stride[next] == stride[prev] * extent[prev]): always
// true for a whole tensor; a slab of a label in the middle of a run (the
// streamed paths lower slabs with the whole tensor's strides) breaks it there.
template <typename Pred>
std::vector<std::vector<int>> runs(const Side& s, Pred in) {
  std::vector<std::vector<int>> out;
  bool open = false;
  int prev = -1;
  for (int id : s.modes) {
    if (in(id)) {
      const bool chained =
          open && s.stride[static_cast<std::size_t>(id)] ==
                      s.stride[static_cast<std::size_t>(prev)] *
                          s.extent[static_cast<std::size_t>(prev)];
      if (!chained) out.emplace_back();
      out.back().push_back(id);
      open = true;
      prev = id;
    } else {
      open = false;
    }
  }
  return out;
}

std::int64_t product(const ValidatedContraction& v, const std::vector<int>& ids) {
  std::int64_t p = 1;
  for (int id : ids) p *= v.labels[static_cast<std::size_t>(id)].extent;
  return p;
}

// Merge consecutive composite entries that chain (str[i+1] == str[i]*ext[i]).
void push_group(const ValidatedContraction& v, const std::vector<int>& ids,
                const std::vector<std::int64_t>& str_of, std::vector<std::int64_t>& ext,
                std::vector<std::int64_t>& str) {
  for (int id : ids) {
    const std::int64_t e = v.labels[static_cast<std::size_t>(id)].extent;
    const std::int64_t s = str_of[static_cast<std::size_t>(id)];
    if (!ext.empty() && str.back() * ext.back() == s) {
      ext.back() *= e;
      continue;
    }
    ext.push_back(e);
    str.push_back(s);
  }
  if (ext.empty()) {
    ext.push_back(1);
    str.push_back(0);
  }
}

// Sub-indices of a group: consecutive labels merged where they chain in
// every operand they address (stride[next] == stride[prev] * extent[prev]).
struct SubIdx {
  std::vector<std::int64_t> ext, sa, sb;
};
SubIdx sub_indices(const ValidatedContraction& v, const std::vector<int>& ids,
                   const std::vector<std::int64_t>& sa, const std::vector<std::int64_t>& sb,
                   bool use_a, bool use_b) {
  SubIdx g;
  for (int id : ids) {
    const std::int64_t e = v.labels[static_cast<std::size_t>(id)].extent;
    const std::int64_t a = sa[static_cast<std::size_t>(id)], b = sb[static_cast<std::size_t>(id)];
    if (!g.ext.empty() && (!use_a || g.sa.back() * g.ext.back() == a) &&
        (!use_b || g.sb.back() * g.ext.back() == b)) {
      g.ext.back() *= e;
      continue;
    }
    g.ext.push_back(e);
    g.sa.push_back(use_a ? a : 0);
    g.sb.push_back(use_b ? b : 0);
  }
  return g;
}

// Can one operand's tensor map carry (outer group, k group)? Mirrors the
// box rules of make_map (device/gemm_dmma.cu): the unit-stride sub-index
// leads; k's inner sub-index is boxed 16; the outer index is spanned 128 at a
// time (K-major) or split as (outer % 16, outer / 16) with the 8 chunks of a
// tile spanned (MN-major). A span covers a sub-index whose extent it divides
// (or is a multiple of) and may continue into the next; at most 5 dims, even
// strides (16-byte multiples), extents below 2^31.
bool fits_map(const std::vector<std::int64_t>& oe, const std::vector<std::int64_t>& os,
              const std::vector<std::int64_t>& ke, const std::vector<std::int64_t>& ks) {
  if (oe.empty() || ke.empty()) return false;
  const bool kmajor = os[0] != 1;
  if (kmajor && ks[0] != 1) return false;
  if (ke.size() > 1 && ke[0] % 16) return false;
  // span rule over group g (first sub-index g0) covering `span` values
  auto spans = [](std::vector<std::int64_t> g, std::int64_t span) {
    if (g.size() == 1 || g[0] % span == 0) return true;
    if (span % g[0]) return false;
    return g.size() <= 2 || g[1] % (span / g[0]) == 0;
  };
  std::size_t dims = 0;
  if (kmajor) {
    if (!spans(oe, 128)) return false;
    dims = 1 + oe.size() + (ke.size() - 1);
  } else {
    if (oe.size() > 1 && oe[0] % 16) return false;
    if (oe[0] % 16 == 0) {
      std::vector<std::int64_t> hi(oe);
      hi[0] /= 16;
      if (hi[0] == 1 && hi.size() > 1) hi.erase(hi.begin());
      if (!spans(hi, 8)) return false;
      dims = 2 + hi.size() + (ke.size() - 1);
    } else {
      dims = 2 + (ke.size() - 1);  // plain: eight 16 x 16 boxes
    }
  }
  if (dims > 5) return false;
  auto strides_ok = [](const std::vector<std::int64_t>& e, const std::vector<std::int64_t>& s,
                       bool lead) {
    for (std::size_t i = 0; i < e.size(); ++i) {
      if (e[i] >= (1LL << 31)) return false;
      if (lead && i == 0) continue;
      if (e[i] > 1 && (s[i] <= 0 || s[i] % 2 || s[i] * 8 >= (1LL << 40))) return false;
    }
    return true;
  };
  return strides_ok(oe, os, !kmajor) && strides_ok(ke, ks, kmajor);
}

// The L4 recipe, or false when the groups do not fit the tensor maps.
bool lower_groups(const ValidatedContraction& v, const Side& A, const Side& B,
                  const std::vector<std::int64_t>& ostr, DeviceRecipe& r) {
  auto is_k = [&](int id) { return v.labels[static_cast<std::size_t>(id)].contracted; };
  if (A.modes.empty() || B.modes.empty()) return false;
  const int ua = A.modes[0], ub = B.modes[0];
  std::vector<int> kl, ml, nl;
  for (int id : A.modes) (is_k(id) ? kl : ml).push_back(id);
  for (int id : B.modes)
    if (!is_k(id)) nl.push_back(id);
  if (kl.empty() || ml.empty() || nl.empty()) return false;
  // k's inner sub-index: the unit-stride label of a K-major operand (both
  // K-major on different labels = class 3.1: no common order, permute)
  int kin = -1;
  if (is_k(ua) && is_k(ub) && ua != ub) return false;
  if (is_k(ua)) kin = ua;
  else if (is_k(ub)) kin = ub;
  else {
    kin = kl[0];
    for (int id : kl)
      if (v.labels[static_cast<std::size_t>(id)].extent % 16 == 0) {
        kin = id;
        break;
      }
  }
  std::vector<int> korder{kin};
  for (int id : kl)
    if (id != kin) korder.push_back(id);
  const SubIdx K = sub_indices(v, korder, A.stride, B.stride, true, true);
  const SubIdx M = sub_indices(v, ml, A.stride, B.stride, true, false);
  const SubIdx N = sub_indices(v, nl, A.stride, B.stride, false, true);
  if (K.ext.size() > TCB_MAX_DIMS || M.ext.size() > TCB_MAX_DIMS || N.ext.size() > TCB_MAX_DIMS)
    return false;
  if (!fits_map(M.ext, M.sa, K.ext, K.sa) || !fits_map(N.ext, N.sb, K.ext, K.sb)) return false;
  r.m = product(v, ml);
  r.n = product(v, nl);
  r.k = product(v, korder);
  if (r.m < 2 || r.n < 2) return false;  // GEMV shapes take the plain strides
  r.a_sm = M.sa[0];
  r.a_sk = K.sa[0];
  r.b_sk = K.sb[0];
  r.b_sn = N.sb[0];
  r.gm_ext = M.ext;
  r.gm_sa = M.sa;
  r.gn_ext = N.ext;
  r.gn_sb = N.sb;
  r.gk_ext = K.ext;
  r.gk_sa = K.sa;
  r.gk_sb = K.sb;
  push_group(v, ml, ostr, r.row_ext, r.row_str);
  push_group(v, nl, ostr, r.col_ext, r.col_str);
  r.layout = "L4";
  return true;
}

}  // namespace

std::string DeviceRecipe::summary() const {
  std::ostringstream os;
  os << layout << " gemm m=" << m << " n=" << n << " k=" << k;
  if (layout == "L4") {
    auto grp = [&](const char* name, const std::vector<std::int64_t>& e,
                   const std::vector<std::int64_t>& s1, const std::vector<std::int64_t>* s2) {
      os << ' ' << name << '[';
      for (std::size_t i = 0; i < e.size(); ++i) {
        os << (i ? "," : "") << e[i] << ':' << s1[i];
        if (s2) os << '/' << (*s2)[i];
      }
      os << ']';
    };
    grp("m", gm_ext, gm_sa, nullptr);
    grp("n", gn_ext, gn_sb, nullptr);
    grp("k", gk_ext, gk_sa, &gk_sb);
    os << " batch=[] permutes=0";
    return os.str();
  }
  os << " a(" << a_sm << "," << a_sk << ") b(" << b_sk << "," << b_sn << ") batch=[";
  for (std::size_t i = 0; i < bat_ext.size(); ++i) os << (i ? "," : "") << bat_ext[i];
  os << "] permutes=" << permutes.size();
  return os.str();
}

DeviceRecipe lower(const ValidatedContraction& v, bool index_groups,
                   const ValidatedContraction* layout) {
  // TC_INDEX_GROUPS=0 disables L4 (A/B comparisons against L3)
  if (const char* env = std::getenv("TC_INDEX_GROUPS"); env != nullptr && env[0] == '0')
    index_groups = false;
  const ValidatedContraction& lay = layout ? *layout : v;
  const std::size_t nlab = v.labels.size();
  Side A = side_of(v, lay, false), B = side_of(v, lay, true);
  std::vector<std::int64_t> ostr(nlab, 0);
  {
    std::int64_t run = 1;
    for (const auto& ix : v.spec.output.indices) {
      const int id = v.label_index(ix.label);
      ostr[static_cast<std::size_t>(id)] = run;
      run *= lay.labels[static_cast<std::size_t>(id)].extent;
    }
  }
  auto is_k = [&](int id) { return v.labels[static_cast<std::size_t>(id)].contracted; };
  auto is_free = [&](int id) { return !v.labels[static_cast<std::size_t>(id)].contracted; };

  const auto ka = runs(A, is_k), kb = runs(B, is_k);
  const bool a_ok = ka.size() <= 1, b_ok = kb.size() <= 1;
  const std::vector<int> ka_order = ka.empty() ? std::vector<int>{} : ka[0];
  const std::vector<int> kb_order = kb.empty() ? std::vector<int>{} : kb[0];

  // Decide which operands are permuted and the common K order.
  bool perm_a = false, perm_b = false;
  std::vector<int> korder;
  auto mode_order_k = [&](const Side& s) {
    std::vector<int> o;
    for (int id : s.modes)
      if (is_k(id)) o.push_back(id);
    return o;
  };
  if (a_ok && b_ok) {
    if (ka_order == kb_order) {
      korder = ka_order;
    } else if (A.elements <= B.elements) {
      perm_a = true;
      korder = kb_order;
    } else {
      perm_b = true;
      korder = ka_order;
    }
  } else if (a_ok) {
    perm_b = true;
    korder = ka_order;
  } else if (b_ok) {
    perm_a = true;
    korder = kb_order;
  } else {
    perm_a = perm_b = true;
    const bool b_lead_k = !B.modes.empty() && is_k(B.modes[0]);
    korder = b_lead_k ? mode_order_k(B) : mode_order_k(A);
  }

  DeviceRecipe r;
  if ((perm_a || perm_b) && index_groups && lower_groups(v, A, B, ostr, r)) return r;
  r = DeviceRecipe{};
  r.k = product(v, korder);
  std::vector<int> mgroup, ngroup, batch;

  // ---- left operand
  if (perm_a) {
    std::vector<int> frees;
    for (int id : A.modes)
      if (is_free(id)) frees.push_back(id);
    const bool free_first = A.modes.empty() || is_free(A.modes[0]);
    std::vector<int> order = free_first ? frees : korder;
    const std::vector<int>& tail = free_first ? korder : frees;
    order.insert(order.end(), tail.begin(), tail.end());
    PermuteStep ps;
    ps.right = false;
    std::vector<std::int64_t> dense(nlab, 0);
    std::int64_t run = 1;
    for (int id : order) {
      ps.ext.push_back(v.labels[static_cast<std::size_t>(id)].extent);
      ps.src_str.push_back(A.stride[static_cast<std::size_t>(id)]);
      dense[static_cast<std::size_t>(id)] = run;
      run *= v.labels[static_cast<std::size_t>(id)].extent;
    }
    ps.elements = run;
    r.permutes.push_back(ps);
    A.stride = dense;
    mgroup = frees;
  } else {
    const auto mr = runs(A, is_free);
    // the M group is the run holding the unit-stride label if that is free,
    // else the largest run; the other free runs become batch dimensions
    std::size_t pick = 0;
    if (!mr.empty()) {
      if (!(is_free(A.modes[0]))) {
        for (std::size_t i = 1; i < mr.size(); ++i)
          if (product(v, mr[i]) > product(v, mr[pick])) pick = i;
      }
      mgroup = mr[pick];
      for (std::size_t i = 0; i < mr.size(); ++i)
        if (i != pick) batch.insert(batch.end(), mr[i].begin(), mr[i].end());
    }
  }
  // ---- right operand
  if (perm_b) {
    std::vector<int> frees;
    for (int id : B.modes)
      if (is_free(id)) frees.push_back(id);
    const bool k_first = !B.modes.empty() && is_k(B.modes[0]);
    std::vector<int> order = k_first ? korder : frees;
    const std::vector<int>& tail = k_first ? frees : korder;
    order.insert(order.end(), tail.begin(), tail.end());
    PermuteStep ps;
    ps.right = true;
    std::vector<std::int64_t> dense(nlab, 0);
    std::int64_t run = 1;
    for (int id : order) {
      ps.ext.push_back(v.labels[static_cast<std::size_t>(id)].extent);
      ps.src_str.push_back(B.stride[static_cast<std::size_t>(id)]);
      dense[static_cast<std::size_t>(id)] = run;
      run *= v.labels[static_cast<std::size_t>(id)].extent;
    }
    ps.elements = run;
    r.permutes.push_back(ps);
    B.stride = dense;
    ngroup = frees;
  } else {
    const auto nr = runs(B, is_free);
    std::size_t pick = 0;
    if (!nr.empty()) {
      if (!is_free(B.modes[0])) {
        for (std::size_t i = 1; i < nr.size(); ++i)
          if (product(v, nr[i]) > product(v, nr[pick])) pick = i;
      }
      ngroup = nr[pick];
      for (std::size_t i = 0; i < nr.size(); ++i)
        if (i != pick) batch.insert(batch.end(), nr[i].begin(), nr[i].end());
    }
  }

  r.m = product(v, mgroup);
  r.n = product(v, ngroup);
  auto first_stride = [](const std::vector<int>& g, const std::vector<std::int64_t>& s) {
    return g.empty() ? std::int64_t{1} : s[static_cast<std::size_t>(g[0])];
  };
  r.a_sm = first_stride(mgroup, A.stride);
  r.a_sk = first_stride(korder, A.stride);
  r.b_sk = first_stride(korder, B.stride);
  r.b_sn = first_stride(ngroup, B.stride);
  push_group(v, mgroup, ostr, r.row_ext, r.row_str);
  push_group(v, ngroup, ostr, r.col_ext, r.col_str);
  for (int id : batch) {
    r.bat_ext.push_back(v.labels[static_cast<std::size_t>(id)].extent);
    r.bat_sa.push_back(A.stride[static_cast<std::size_t>(id)]);
    r.bat_sb.push_back(B.stride[static_cast<std::size_t>(id)]);
    r.bat_sc.push_back(ostr[static_cast<std::size_t>(id)]);
  }
  r.layout = !r.permutes.empty() ? "L3" : (batch.empty() ? "L1" : "L2");
  return r;
}

}  // namespace tc
