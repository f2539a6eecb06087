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
// The output is never permuted: the GEMM epilogue addresses C through the
// composite row (M labels) and column (N labels) strides. Extent-1 labels are
// dropped first (any coordinate of them is 0).
#include <algorithm>
#include <numeric>
#include <sstream>

#include "tc/contract.hpp"

namespace tc {
namespace {

struct Side {
  std::vector<int> modes;              // non-unit label ids in mode order
  std::vector<std::int64_t> stride;    // per label id (canonical), 0 if absent
  std::int64_t elements = 1;
};

Side side_of(const ValidatedContraction& v, bool right) {
  Side s;
  s.stride.assign(v.labels.size(), 0);
  const int rank = right ? v.right_rank() : v.left_rank();
  std::int64_t run = 1;
  for (int m = 0; m < rank; ++m) {
    const LabelInfo& li = right ? v.label_at_right_mode(m) : v.label_at_left_mode(m);
    const int id = v.label_index(li.label);
    s.stride[static_cast<std::size_t>(id)] = run;
    run *= li.extent;
    if (li.extent > 1) s.modes.push_back(id);
  }
  s.elements = run;
  return s;
}

// Maximal runs of consecutive (non-unit) modes whose labels satisfy `in`.
template <typename Pred>
std::vector<std::vector<int>> runs(const Side& s, Pred in) {
  std::vector<std::vector<int>> out;
  bool open = false;
  for (int id : s.modes) {
    if (in(id)) {
      if (!open) out.emplace_back();
      out.back().push_back(id);
      open = true;
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

}  // namespace

std::string DeviceRecipe::summary() const {
  std::ostringstream os;
  os << layout << " gemm m=" << m << " n=" << n << " k=" << k << " a(" << a_sm << "," << a_sk
     << ") b(" << b_sk << "," << b_sn << ") batch=[";
  for (std::size_t i = 0; i < bat_ext.size(); ++i) os << (i ? "," : "") << bat_ext[i];
  os << "] permutes=" << permutes.size();
  return os.str();
}

DeviceRecipe lower(const ValidatedContraction& v) {
  const std::size_t nlab = v.labels.size();
  Side A = side_of(v, false), B = side_of(v, true);
  std::vector<std::int64_t> ostr(nlab, 0);
  {
    std::int64_t run = 1;
    for (const auto& ix : v.spec.output.indices) {
      const int id = v.label_index(ix.label);
      ostr[static_cast<std::size_t>(id)] = run;
      run *= v.labels[static_cast<std::size_t>(id)].extent;
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
