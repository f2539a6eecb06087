// k4 — level-2/1 recipes: GEMV and DOT (the reference's class-2 and class-1
// kernels: ReferenceBackend::gemv/dot, src/kernels_reference.cpp:81-120 and
// :140-149, driven by the executor's GEMV and DOT loops, src/executor.cpp:
// 181-227). Both are HBM-bound (~8 B per FMA), so the design goal is
// coalescing and bytes in flight.
//
// Canonical summation order (shared by every kernel below, so results are
// bit-reproducible and independent of the operand layout — cf. the
// reference's transpose-equivalence test, tests/test_kernels.cpp:86-116):
//   K is cut into chunks of `chunk` (a multiple of 64); inside a chunk, k-lane
//   λ = (k - k0) mod 64 accumulates its terms in increasing k; the 64 lane
//   sums are paired (2j, 2j+1) and the 32 pairs combined by a fixed xor tree;
//   chunk results are summed in chunk order by a 256-thread fixed tree.
//   * K-major matrix (k contiguous): one warp per (row, chunk); lane l owns
//     k-lanes 2l, 2l+1 and streams them with 16-byte loads, 4 in flight;
//   * row-contiguous matrix: warps cover 32-64 rows (16-byte loads) or, for
//     short matrices, several columns per access; each thread owns up to 8
//     k-lanes (8 loads in flight), combined through shared memory with the
//     same tree;
//   * DOT is the one-row case of the K-major kernel.
#include <algorithm>

#include "tcb_internal.cuh"

namespace tcb {
namespace {

struct GvParams {
  const double* M;  // matrix(o, k) at M + off_m(b) + o*so + k*sk
  const double* v;  // vector(k) at v + off_v(b) + k*sv
  double* y;        // y(o) at y + off_y(b) + composite(o)
  int64_t rows, K, so, sk, sv;
  int ny;
  int64_t y_ext[TCB_MAX_DIMS], y_str[TCB_MAX_DIMS];
  int nbatch;
  int64_t bat_ext[TCB_MAX_DIMS], bat_sm[TCB_MAX_DIMS], bat_sv[TCB_MAX_DIMS], bat_sy[TCB_MAX_DIMS];
  int64_t batch;
  double alpha, beta;
  int splits;
  int64_t chunk;  // k per split, a multiple of 64
  bool vec;       // 16-byte loads legal (k-major kernel)
  double* ws;     // partials [(b*rows + o)*splits + s]
};

__device__ __forceinline__ void gv_batch(const GvParams& p, int64_t b, int64_t& om, int64_t& ov,
                                         int64_t& oy) {
  om = ov = oy = 0;
  for (int i = 0; i < p.nbatch; ++i) {
    const int64_t c = b % p.bat_ext[i];
    b /= p.bat_ext[i];
    om += c * p.bat_sm[i];
    ov += c * p.bat_sv[i];
    oy += c * p.bat_sy[i];
  }
}

__device__ __forceinline__ int64_t gv_row(const GvParams& p, int64_t o) {
  int64_t off = 0;
  for (int i = 0; i < p.ny - 1; ++i) {
    off += (o % p.y_ext[i]) * p.y_str[i];
    o /= p.y_ext[i];
  }
  return off + o * p.y_str[p.ny - 1];
}

__device__ __forceinline__ void gv_store(const GvParams& p, int64_t b, int64_t o, int s,
                                         double sum) {
  if (p.splits > 1) {
    p.ws[(b * p.rows + o) * p.splits + s] = sum;
    return;
  }
  int64_t om, ov, oy;
  gv_batch(p, b, om, ov, oy);
  double* dst = p.y + oy + gv_row(p, o);
  double r = p.alpha * sum;
  if (p.beta != 0.0) r += p.beta * *dst;
  *dst = r;
}

// one warp per (batch, row, split); lane l owns k-lanes 2l and 2l+1
__global__ void __launch_bounds__(256) gemv_kmajor(GvParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t items = p.batch * p.rows * p.splits;
  for (int64_t it = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
       it < items; it += nwarps) {
    const int s = static_cast<int>(it % p.splits);
    const int64_t o = (it / p.splits) % p.rows;
    const int64_t b = it / (p.splits * p.rows);
    int64_t om, ov, oy;
    gv_batch(p, b, om, ov, oy);
    const double* mrow = p.M + om + o * p.so;
    const double* vec = p.v + ov;
    const int64_t k0 = s * p.chunk, k1 = min(p.K, k0 + p.chunk);
    double e0 = 0.0, e1 = 0.0;  // k-lanes 2l, 2l+1
    if (p.vec) {
      // k0 is a multiple of 64 and rows/vector 16-byte aligned (checked on host)
      const int64_t full = k0 + ((k1 - k0) / 64) * 64;
      int64_t k = k0 + 2 * lane;
#pragma unroll 4
      for (; k < full; k += 64) {
        const double2 a = __ldcs(reinterpret_cast<const double2*>(mrow + k));
        const double2 x = __ldg(reinterpret_cast<const double2*>(vec + k));
        e0 = fma(a.x, x.x, e0);
        e1 = fma(a.y, x.y, e1);
      }
      if (k < k1) e0 = fma(__ldcs(mrow + k), __ldg(vec + k), e0);
      if (k + 1 < k1) e1 = fma(__ldcs(mrow + k + 1), __ldg(vec + k + 1), e1);
    } else {
#pragma unroll 4
      for (int64_t k = k0 + 2 * lane; k < k1; k += 64) {
        e0 = fma(__ldg(mrow + k * p.sk), __ldg(vec + k * p.sv), e0);
        if (k + 1 < k1) e1 = fma(__ldg(mrow + (k + 1) * p.sk), __ldg(vec + (k + 1) * p.sv), e1);
      }
    }
    double acc = e0 + e1;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) gv_store(p, b, o, s, acc);
  }
}

// Row-contiguous matrix, 16 warps per block. A warp covers RL*VR consecutive
// rows x G = 32/RL consecutive columns, where RL (<= 32) is the number of lanes
// along rows (fewer than 32 when the matrix has few rows: short-wide matrices
// still get 128-256-byte warp accesses). Lane (r, c) owns rows r*VR..r*VR+VR-1
// (16-byte loads when VR == 2) and, with the warp index ty, the k-lanes
// c + G*ty + 16G*j (j < NJ = 4/G) of the canonical 64-lane order. The loads
// of DEPTH 64-column steps are in flight at once (DEPTH*NJ*VR doubles per
// thread). Lane sums meet in shared memory and are combined with the same
// tree as gemv_kmajor.
// The canonical combination of the 64 k-lane sums of one row (column rr of
// red): pairs (2j, 2j+1), then the xor tree of gemv_kmajor's shuffles —
// T(lo, step, n) = T(lo, 2 step, n/2) + T(lo + step, 2 step, n/2) — evaluated
// depth first so only ~log2(32) partial sums are live.
template <int LO, int STEP, int N>
__device__ __forceinline__ double lane_tree(const double (*red)[64 + 1], int rr) {
  if constexpr (N == 1) {
    return red[2 * LO][rr] + red[2 * LO + 1][rr];
  } else {
    const double a = lane_tree<LO, 2 * STEP, N / 2>(red, rr);
    return a + lane_tree<LO + STEP, 2 * STEP, N / 2>(red, rr);
  }
}

template <int VR, int G>
__global__ void __launch_bounds__(512, 2) gemv_omajor(GvParams p) {
  constexpr int RL = 32 / G, NJ = 4 / G, DEPTH = 2;
  __shared__ double red[64][64 + 1];
  const int lane = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int r = lane % RL, c = lane / RL;
  constexpr int rows_per_tile = RL * VR;
  const int64_t rblocks = (p.rows + rows_per_tile - 1) / rows_per_tile;
  const int64_t items = p.batch * rblocks * p.splits;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int s = static_cast<int>(it % p.splits);
    const int64_t rb = (it / p.splits) % rblocks;
    const int64_t b = it / (p.splits * rblocks);
    int64_t om, ov, oy;
    gv_batch(p, b, om, ov, oy);
    const int64_t o = rb * rows_per_tile + r * VR;  // first row of this lane
    const int64_t k0 = s * p.chunk, k1 = min(p.K, k0 + p.chunk);
    double acc[NJ][VR];
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int v = 0; v < VR; ++v) acc[j][v] = 0.0;
    if (o < p.rows) {
      const double* mcol = p.M + om + o * p.so;
      const double* vec = p.v + ov;
      const int kl = c + G * ty;  // this thread's first k-lane
#pragma unroll 1
      for (int64_t kb = k0; kb < k1; kb += 64 * DEPTH) {
        double a[DEPTH][NJ][VR], x[DEPTH][NJ];
#pragma unroll
        for (int d = 0; d < DEPTH; ++d)
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            const int64_t k = kb + 64 * d + kl + 16 * G * j;
            const bool ok = k < k1;
            x[d][j] = ok ? __ldg(vec + k * p.sv) : 0.0;
            if (VR == 2) {
              const double2 t = ok ? __ldcs(reinterpret_cast<const double2*>(mcol + k * p.sk))
                                   : make_double2(0.0, 0.0);
              a[d][j][0] = t.x;
              a[d][j][VR - 1] = t.y;
            } else {
              a[d][j][0] = ok ? __ldcs(mcol + k * p.sk) : 0.0;
            }
          }
        // in increasing k per k-lane; out-of-range terms are skipped (not
        // added as zeros) so the FMA chain matches the canonical order exactly
#pragma unroll
        for (int d = 0; d < DEPTH; ++d)
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            if (kb + 64 * d + kl + 16 * G * j < k1)
#pragma unroll
              for (int v = 0; v < VR; ++v) acc[j][v] = fma(a[d][j][v], x[d][j], acc[j][v]);
      }
    }
    // red[lambda][row in tile]
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int v = 0; v < VR; ++v) red[c + G * (ty + 16 * j)][r * VR + v] = acc[j][v];
    __syncthreads();
    for (int rr = threadIdx.x; rr < rows_per_tile; rr += blockDim.x) {
      const int64_t orow = rb * rows_per_tile + rr;
      if (orow >= p.rows) continue;
      gv_store(p, b, orow, s, lane_tree<0, 1, 32>(red, rr));
    }
    __syncthreads();
  }
}

// chunk partials of one output -> y, summed by a fixed 256-thread tree
__global__ void __launch_bounds__(256) gemv_finalize(GvParams p) {
  __shared__ double red[256];
  const int64_t n = p.batch * p.rows;
  for (int64_t e = blockIdx.x; e < n; e += gridDim.x) {
    const double* part = p.ws + e * p.splits;
    double sum = 0.0;
    for (int s = threadIdx.x; s < p.splits; s += 256) sum += part[s];
    red[threadIdx.x] = sum;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
      if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const int64_t o = e % p.rows, b = e / p.rows;
      int64_t om, ov, oy;
      gv_batch(p, b, om, ov, oy);
      double* dst = p.y + oy + gv_row(p, o);
      double r = p.alpha * red[0];
      if (p.beta != 0.0) r += p.beta * *dst;
      *dst = r;
    }
    __syncthreads();
  }
}

}  // namespace

// d has m == 1 or n == 1 (or both: DOT).
int launch_gemv(const tcb_gemm_desc& d, const double* A, const double* B, double* C) {
  ThreadState& st = state();
  GvParams p{};
  const bool rows_are_m = d.n == 1;  // y = A x  (else y^T = a^T B)
  if (rows_are_m) {
    p.M = A;
    p.v = B;
    p.rows = d.m;
    p.so = d.a_sm;
    p.sk = d.a_sk;
    p.sv = d.b_sk;
    p.ny = d.c_nrow;
    for (int i = 0; i < TCB_MAX_DIMS; ++i) {
      p.y_ext[i] = d.c_row_ext[i];
      p.y_str[i] = d.c_row_str[i];
      p.bat_sm[i] = d.bat_sa[i];
      p.bat_sv[i] = d.bat_sb[i];
    }
  } else {
    p.M = B;
    p.v = A;
    p.rows = d.n;
    p.so = d.b_sn;
    p.sk = d.b_sk;
    p.sv = d.a_sk;
    p.ny = d.c_ncol;
    for (int i = 0; i < TCB_MAX_DIMS; ++i) {
      p.y_ext[i] = d.c_col_ext[i];
      p.y_str[i] = d.c_col_str[i];
      p.bat_sm[i] = d.bat_sb[i];
      p.bat_sv[i] = d.bat_sa[i];
    }
  }
  p.y = C;
  p.K = d.k;
  p.nbatch = d.nbatch;
  p.batch = 1;
  for (int i = 0; i < TCB_MAX_DIMS; ++i) {
    p.bat_ext[i] = d.bat_ext[i];
    p.bat_sy[i] = d.bat_sc[i];
  }
  for (int i = 0; i < d.nbatch; ++i) p.batch *= d.bat_ext[i];
  p.alpha = d.alpha;
  p.beta = d.beta;
  const int sms = num_sms();
  // the k-contiguous kernel when rows are not unit-stride or there is one row
  const bool use_k = p.rows == 1 || (p.sk == 1 && p.so != 1) || (p.so != 1 && p.sk != 1);

  // Chunking depends only on (batch*rows, K) — never on the kernel — and
  // chunks are multiples of 64, so the summation order is layout-free.
  const int64_t rows_total = p.batch * p.rows;
  // enough (row, chunk) items for several waves of either kernel
  const int64_t target = static_cast<int64_t>(sms) * 2048;
  int64_t splits = 1;
  if (rows_total < target)
    splits = std::min<int64_t>((target + rows_total - 1) / rows_total,
                               std::max<int64_t>(1, d.k / 1024));
  splits = std::max<int64_t>(1, std::min<int64_t>(splits, 65536));
  p.chunk = ((d.k + splits - 1) / splits + 63) / 64 * 64;
  splits = (d.k + p.chunk - 1) / p.chunk;
  p.splits = static_cast<int>(splits);

  // 16-byte loads: unit k-stride, 16-byte aligned row/vector starts
  bool vec = p.sk == 1 && p.sv == 1 && reinterpret_cast<uintptr_t>(p.M) % 16 == 0 &&
             reinterpret_cast<uintptr_t>(p.v) % 16 == 0 && (p.rows == 1 || p.so % 2 == 0);
  for (int i = 0; i < d.nbatch && vec; ++i) vec = p.bat_sm[i] % 2 == 0 && p.bat_sv[i] % 2 == 0;
  p.vec = vec;

  if (splits > 1) {
    const int64_t need = rows_total * splits * 8;
    if (need > st.ws_bytes) {
      if (st.ws) cudaFree(st.ws);
      st.ws = nullptr;
      st.ws_bytes = 0;
      TCB_CUDA(cudaMalloc(&st.ws, need));
      st.ws_bytes = need;
    }
    p.ws = static_cast<double*>(st.ws);
  }
  int launches = 0;
  if (use_k) {
    const int64_t warps = rows_total * splits;
    const int blocks = static_cast<int>(std::min<int64_t>((warps + 7) / 8, sms * 32LL));
    gemv_kmajor<<<blocks, 256, 0, st.stream>>>(p);
  } else {
    // lanes along rows: fewer than 32 for short matrices (then each warp
    // access spans several columns); 2 rows per lane when 16-byte loads are legal
    int RL = 32;
    while (RL > 1 && RL / 2 >= p.rows) RL /= 2;
    if (RL < 8) RL = 8;  // G = 32/RL must divide 4
    bool vr2 = p.rows % 2 == 0 && p.so == 1 && p.sk % 2 == 0 &&
               reinterpret_cast<uintptr_t>(p.M) % 16 == 0;
    for (int i = 0; i < d.nbatch && vr2; ++i) vr2 = p.bat_sm[i] % 2 == 0;
    // two rows per lane: half the lanes along rows when that still covers them
    if (vr2 && p.rows < 2 * RL) {
      if (RL > 8) RL /= 2;
      else vr2 = false;
    }
    const int g = 32 / RL;
    const int per_tile = RL * (vr2 ? 2 : 1);
    const int64_t items = p.batch * ((p.rows + per_tile - 1) / per_tile) * splits;
    const int blocks = static_cast<int>(std::min<int64_t>(items, sms * 8LL));
    auto kern = vr2 ? (g == 1 ? gemv_omajor<2, 1> : g == 2 ? gemv_omajor<2, 2> : gemv_omajor<2, 4>)
                    : (g == 1 ? gemv_omajor<1, 1> : g == 2 ? gemv_omajor<1, 2> : gemv_omajor<1, 4>);
    kern<<<blocks, 512, 0, st.stream>>>(p);
  }
  TCB_LAUNCHED();
  ++launches;
  if (splits > 1) {
    const int blocks = static_cast<int>(std::min<int64_t>(rows_total, sms * 16LL));
    gemv_finalize<<<blocks, 256, 0, st.stream>>>(p);
    TCB_LAUNCHED();
    ++launches;
  }
  st.last_info.path = (d.m == 1 && d.n == 1) ? 3 : 2;
  st.last_info.splits = p.splits;
  st.last_info.units = rows_total * splits;
  st.last_info.grid = 0;
  st.last_info.launches = launches;
  return TCB_OK;
}

}  // namespace tcb
