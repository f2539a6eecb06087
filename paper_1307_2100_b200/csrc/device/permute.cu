// k3 — operand permutation (the COPY of the reference's COPY+GEMM).
//
// The reference packs every strided 2-mode slice into a contiguous buffer on
// the CPU, once per kernel call (materialize, src/executor.cpp:41-59; also
// pack_slice, src/tensor.cpp:150-171). Here a whole operand is re-laid out once
// per contraction, HBM-bound, in one launch:
//   * same unit-stride dim in source and destination -> run copy: one warp per
//     contiguous run, 16-byte vector loads/stores when aligned;
//   * different unit-stride dims -> 32x32 shared-memory tiled transpose
//     (padded, conflict-free), remaining dims on the grid;
//   * no unit-stride source dim -> element-wise gather (rare, small).
// Dimensions are first simplified: extent-1 dims dropped, dims that are
// contiguous in both layouts merged.
#include <algorithm>
#include <vector>

#include "tcb_internal.cuh"

namespace tcb {
namespace {

constexpr int MAXR = 8;

struct PermParams {
  int rank;                 // after simplification
  int64_t ext[MAXR];        // destination order, first fastest
  int64_t sstr[MAXR];       // source strides per dim
  int64_t dstr[MAXR];       // destination strides (dense)
  int t;                    // transpose: the source unit-stride dim
  int64_t rows;             // run copy: number of runs / transpose: number of outer slabs
  int outer_n;              // dims enumerated by the grid (all but 0 [and t])
  int outer_dim[MAXR];
};

__device__ __forceinline__ void outer_offsets(const PermParams& p, int64_t idx, int64_t& so,
                                              int64_t& dof) {
  so = 0;
  dof = 0;
  for (int i = 0; i < p.outer_n; ++i) {
    const int d = p.outer_dim[i];
    const int64_t c = idx % p.ext[d];
    idx /= p.ext[d];
    so += c * p.sstr[d];
    dof += c * p.dstr[d];
  }
}

// Same unit-stride dim: copy runs of ext[0] contiguous doubles.
template <bool VEC>
__global__ void perm_runs(PermParams p, const double* __restrict__ src, double* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t L = p.ext[0];
  for (int64_t row = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
       row < p.rows; row += warps) {
    int64_t so, dof;
    outer_offsets(p, row, so, dof);
    const double* s = src + so;
    double* d = dst + dof;
    if (VEC) {
      const double2* s2 = reinterpret_cast<const double2*>(s);
      double2* d2 = reinterpret_cast<double2*>(d);
      for (int64_t i = lane; i < L / 2; i += 32) __stcs(d2 + i, __ldcs(s2 + i));
    } else {
      for (int64_t i = lane; i < L; i += 32) __stcs(d + i, __ldcs(s + i));
    }
  }
}

// Different unit-stride dims: transpose tiles of (dst dim 0) x (src dim t).
__global__ void perm_transpose(PermParams p, const double* __restrict__ src,
                               double* __restrict__ dst) {
  __shared__ double tile[32][33];
  const int64_t e0 = p.ext[0], et = p.ext[p.t];
  const int64_t t0n = (e0 + 31) / 32, ttn = (et + 31) / 32;
  const int64_t tiles = t0n * ttn * p.rows;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int64_t b = blockIdx.x; b < tiles; b += gridDim.x) {
    const int64_t slab = b / (t0n * ttn);
    const int64_t rem = b % (t0n * ttn);
    const int64_t i0 = (rem % t0n) * 32, it = (rem / t0n) * 32;
    int64_t so, dof;
    outer_offsets(p, slab, so, dof);
    // read: consecutive threads along t (unit stride in the source)
    for (int y = ty; y < 32; y += 8) {
      const int64_t a = i0 + y, c = it + tx;
      if (a < e0 && c < et) tile[y][tx] = __ldcs(src + so + a * p.sstr[0] + c);
    }
    __syncthreads();
    // write: consecutive threads along dim 0 (unit stride in the destination)
    for (int y = ty; y < 32; y += 8) {
      const int64_t a = i0 + tx, c = it + y;
      if (a < e0 && c < et) __stcs(dst + dof + a + c * p.dstr[p.t], tile[tx][y]);
    }
    __syncthreads();
  }
}

__global__ void perm_gather(PermParams p, int64_t total, const double* __restrict__ src,
                            double* __restrict__ dst) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t idx = e, so = 0;
    for (int i = 0; i < p.rank; ++i) {
      so += (idx % p.ext[i]) * p.sstr[i];
      idx /= p.ext[i];
    }
    dst[e] = src[so];
  }
}

}  // namespace

int launch_permute(int rank, const int64_t* ext, const int64_t* src_str, const double* src,
                   double* dst) {
  if (rank < 0 || rank > MAXR) return set_error(TCB_EUNSUPPORTED, "permute: rank above 8");
  // simplify: drop extent-1 dims, merge dims contiguous in both layouts
  std::vector<int64_t> e, s;
  int64_t total = 1;
  for (int i = 0; i < rank; ++i) {
    if (ext[i] <= 0) return set_error(TCB_EINVAL, "permute: extent must be positive");
    total *= ext[i];
    if (ext[i] == 1) continue;
    if (!e.empty() && s.back() * e.back() == src_str[i]) {
      e.back() *= ext[i];
      continue;
    }
    e.push_back(ext[i]);
    s.push_back(src_str[i]);
  }
  if (total == 0) return TCB_OK;
  ThreadState& st = state();
  if (e.empty()) {  // a single element
    TCB_CUDA(cudaMemcpyAsync(dst, src, 8, cudaMemcpyDeviceToDevice, st.stream));
    return TCB_OK;
  }
  PermParams p{};
  p.rank = static_cast<int>(e.size());
  int64_t dense = 1;
  for (int i = 0; i < p.rank; ++i) {
    p.ext[i] = e[i];
    p.sstr[i] = s[i];
    p.dstr[i] = dense;
    dense *= e[i];
  }
  const int sms = num_sms();
  if (p.rank == 1 && p.sstr[0] == 1) {
    TCB_CUDA(cudaMemcpyAsync(dst, src, total * 8, cudaMemcpyDeviceToDevice, st.stream));
    return TCB_OK;
  }
  if (p.sstr[0] == 1) {
    p.outer_n = 0;
    for (int i = 1; i < p.rank; ++i) p.outer_dim[p.outer_n++] = i;
    p.rows = total / p.ext[0];
    bool vec = p.ext[0] % 2 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0 &&
               reinterpret_cast<uintptr_t>(dst) % 16 == 0;
    for (int i = 1; i < p.rank && vec; ++i) vec = p.sstr[i] % 2 == 0;
    const int64_t warps_needed = p.rows;
    const int blocks = static_cast<int>(std::min<int64_t>((warps_needed + 7) / 8, sms * 16LL));
    if (vec) perm_runs<true><<<blocks, 256, 0, st.stream>>>(p, src, dst);
    else perm_runs<false><<<blocks, 256, 0, st.stream>>>(p, src, dst);
    TCB_LAUNCHED();
    return TCB_OK;
  }
  int t = -1;
  for (int i = 1; i < p.rank; ++i)
    if (p.sstr[i] == 1) t = i;
  if (t > 0) {
    p.t = t;
    p.outer_n = 0;
    for (int i = 1; i < p.rank; ++i)
      if (i != t) p.outer_dim[p.outer_n++] = i;
    p.rows = total / (p.ext[0] * p.ext[t]);
    const int64_t tiles = ((p.ext[0] + 31) / 32) * ((p.ext[t] + 31) / 32) * p.rows;
    const int blocks = static_cast<int>(std::min<int64_t>(tiles, sms * 8LL));
    perm_transpose<<<blocks, 256, 0, st.stream>>>(p, src, dst);
    TCB_LAUNCHED();
    return TCB_OK;
  }
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, sms * 16LL));
  perm_gather<<<blocks, 256, 0, st.stream>>>(p, total, src, dst);
  TCB_LAUNCHED();
  return TCB_OK;
}

}  // namespace tcb
