// k3 — operand permutation (the COPY of the reference's COPY+GEMM).
//
// The reference packs every strided 2-mode slice into a contiguous buffer on
// the CPU, once per kernel call (materialize, src/executor.cpp:41-59; also
// pack_slice, src/tensor.cpp:150-171). Here a whole operand is re-laid out once
// per contraction, HBM-bound, in one launch:
//   * same unit-stride dim in source and destination -> run copy: blocks walk
//     chunks of contiguous runs (offsets decoded once per block item), 16-byte
//     vectors, 4 in flight per thread;
//   * different unit-stride dims -> 64x64 (large) or 32x64 shared-memory
//     tiled transpose (padded), all loads of a thread in flight before the
//     barrier, remaining dims on the grid;
//   * no unit-stride source dim -> element-wise gather (rare, small).
// Dimensions are first simplified: extent-1 dims dropped, dims that are
// contiguous in both layouts merged.
#include <algorithm>
#include <type_traits>
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
  int t;                    // transpose: the source unit-stride dim; runs: log2(run) or -1
  int64_t runs_per_chunk;   // runs: dim-1 runs handled by one block item
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

// Same unit-stride dim: copy runs of ext[0] contiguous doubles. One block
// per "slab" = all ext[1] runs at one coordinate of the outer dims (decoded
// once per block); inside a slab run r starts at r*sstr[1] (source) and
// r*ext[0] (destination), so no per-element index decoding. Each thread keeps
// UNROLL 16-byte vectors in flight (loads first, then stores).
template <bool VEC>
__global__ void perm_runs(PermParams p, const double* __restrict__ src, double* __restrict__ dst) {
  constexpr int UNROLL = 4;
  using V = typename std::conditional<VEC, double2, double>::type;
  constexpr int W = VEC ? 2 : 1;  // doubles per vector
  const int64_t L = p.ext[0] / W;  // vectors per run
  const int64_t runs = p.rank > 1 ? p.ext[1] : 1;
  const int64_t rpc = p.runs_per_chunk;
  const int64_t chunks = (runs + rpc - 1) / rpc;
  const int lshift = p.t;  // log2(L) when L is a power of two, else -1
  for (int64_t item = blockIdx.x; item < p.rows * chunks; item += gridDim.x) {
    const int64_t slab = item / chunks, r0 = (item % chunks) * rpc;
    const int64_t per_slab = L * min(rpc, runs - r0);
    int64_t so, dof;
    outer_offsets(p, slab, so, dof);
    const int64_t rs = p.rank > 1 ? p.sstr[1] / W : 0;  // run stride in vectors
    const V* s = reinterpret_cast<const V*>(src + so) + r0 * rs;
    V* d = reinterpret_cast<V*>(dst + dof) + r0 * L;
    for (int64_t base = threadIdx.x; base < per_slab; base += blockDim.x * UNROLL) {
      V v[UNROLL];
      int64_t di[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int64_t i = base + u * blockDim.x;
        di[u] = i;
        if (i < per_slab) {
          const int64_t r = lshift >= 0 ? (i >> lshift) : i / L;
          const int64_t c = i - r * L;
          v[u] = __ldcs(s + r * rs + c);
        }
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
        if (di[u] < per_slab) __stcs(d + di[u], v[u]);
    }
  }
}

// Different unit-stride dims: transpose tiles of TA (dst dim 0) x 64 (src
// dim t) through padded shared memory; every thread issues its TA/4 loads
// before the barrier and its TA/4 stores after it (both directions coalesced).
template <int TA>
__global__ void __launch_bounds__(256) perm_transpose(PermParams p, const double* __restrict__ src,
                                                      double* __restrict__ dst) {
  constexpr int NV = TA / 4;  // elements per thread
  __shared__ double tile[TA][65];
  const int64_t e0 = p.ext[0], et = p.ext[p.t];
  const int64_t t0n = (e0 + TA - 1) / TA, ttn = (et + 63) / 64;
  const int64_t tiles = t0n * ttn * p.rows;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int64_t b = blockIdx.x; b < tiles; b += gridDim.x) {
    const int64_t slab = b / (t0n * ttn);
    const int64_t rem = b % (t0n * ttn);
    const int64_t i0 = (rem % t0n) * TA, it = (rem / t0n) * 64;
    int64_t so, dof;
    outer_offsets(p, slab, so, dof);
    double v[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {  // rows y = ty + 8*(j/2), t = it + tx + 32*(j%2)
      const int64_t a = i0 + ty + 8 * (j >> 1), c = it + tx + 32 * (j & 1);
      v[j] = (a < e0 && c < et) ? __ldcs(src + so + a * p.sstr[0] + c) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) tile[ty + 8 * (j >> 1)][tx + 32 * (j & 1)] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NV; ++j) {  // rows a = i0 + tx + 32*(j%(TA/32)), columns c
      constexpr int RA = TA / 32;
      const int ra = tx + 32 * (j % RA), cc = ty + 8 * (j / RA);
      const int64_t a = i0 + ra, c = it + cc;
      if (a < e0 && c < et) __stcs(dst + dof + a + c * p.dstr[p.t], tile[ra][cc]);
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
    note_stream_op();
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
    note_stream_op();
    TCB_CUDA(cudaMemcpyAsync(dst, src, total * 8, cudaMemcpyDeviceToDevice, st.stream));
    return TCB_OK;
  }
  if (p.sstr[0] == 1) {
    // slabs = every coordinate of dims 2.. (dim 1 is walked inside the block)
    p.outer_n = 0;
    for (int i = 2; i < p.rank; ++i) p.outer_dim[p.outer_n++] = i;
    p.rows = total / (p.ext[0] * (p.rank > 1 ? p.ext[1] : 1));
    bool vec = p.ext[0] % 2 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0 &&
               reinterpret_cast<uintptr_t>(dst) % 16 == 0;
    for (int i = 1; i < p.rank && vec; ++i) vec = p.sstr[i] % 2 == 0;
    const int64_t L = p.ext[0] / (vec ? 2 : 1);
    p.t = (L & (L - 1)) == 0 ? __builtin_ctzll(static_cast<unsigned long long>(L)) : -1;
    // ~4096 vectors (32-64 KB) per block item
    const int64_t e1 = p.rank > 1 ? p.ext[1] : 1;
    p.runs_per_chunk = std::max<int64_t>(1, std::min<int64_t>(e1, 4096 / std::max<int64_t>(L, 1)));
    const int64_t items = p.rows * ((e1 + p.runs_per_chunk - 1) / p.runs_per_chunk);
    const int blocks = static_cast<int>(std::min<int64_t>(items, sms * 16LL));
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
    // 64x64 tiles, 4 blocks per SM, once there are >= 8 waves of them
    // (1.07 GB transpose: 0.95 of HBM vs 0.90 with 32x64); smaller (L2-resident)
    // operands keep 32x64 tiles, 8 per SM, for more tiles in flight
    const int64_t slab_tiles64 = ((p.ext[0] + 63) / 64) * ((p.ext[t] + 63) / 64);
    const int ta = slab_tiles64 * p.rows >= sms * 32LL ? 64 : 32;
    const int bps = ta == 64 ? 4 : 8;
    const int64_t tiles = ((p.ext[0] + ta - 1) / ta) * ((p.ext[t] + 63) / 64) * p.rows;
    const int blocks = static_cast<int>(std::min<int64_t>(tiles, sms * static_cast<int64_t>(bps)));
    if (ta == 64) perm_transpose<64><<<blocks, 256, 0, st.stream>>>(p, src, dst);
    else perm_transpose<32><<<blocks, 256, 0, st.stream>>>(p, src, dst);
    TCB_LAUNCHED();
    return TCB_OK;
  }
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, sms * 16LL));
  perm_gather<<<blocks, 256, 0, st.stream>>>(p, total, src, dst);
  TCB_LAUNCHED();
  return TCB_OK;
}

}  // namespace tcb
