// k4 — level-2/1 recipes: GEMV and DOT (the reference's class-2 and class-1
// kernels: ReferenceBackend::gemv/dot, src/kernels_reference.cpp:81-120 and
// :140-149, driven by the executor's GEMV and DOT loops, src/executor.cpp:
// 181-227). Both are HBM-bound (~8-16 B per FMA), so the design goal is
// coalescing and enough bytes in flight:
//   * K-major matrix (k contiguous): one warp per output row and k-chunk,
//     lanes stream k with 8-byte loads, warp-shuffle tree reduction;
//   * row-major-in-outer matrix (rows contiguous): 32 rows x 8 threads per
//     block, coalesced along rows, shared-memory reduction over the k-lanes;
//   * DOT is the one-row case of the K-major kernel.
// Both kernels sum in the same order (32 k-lanes, fixed combine tree) and long
// K is split into 32-multiple chunks summed by a second kernel in chunk order,
// so results are bit-reproducible and independent of the operand layout.
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
  int64_t chunk;   // k per split
  double* ws;      // partials [(b*rows + o)*splits + s]
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

// one warp per (batch, row, split)
__global__ void gemv_kmajor(GvParams p) {
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
    // k-lane l sums k = k0 + l, k0 + l + 32, ... in order; lanes combine in a
    // fixed xor tree. gemv_omajor reproduces exactly this order.
    double acc = 0.0;
#pragma unroll 4
    for (int64_t k = k0 + lane; k < k1; k += 32)
      acc = fma(__ldg(mrow + k * p.sk), __ldg(vec + k * p.sv), acc);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) gv_store(p, b, o, s, acc);
  }
}

// 32 rows x 8 threads per block; rows are the coalesced direction. Thread ty
// carries the 4 k-lanes ty, ty+8, ty+16, ty+24 of the 32-lane order used by
// gemv_kmajor, and the lanes are combined with the same tree, so both layouts
// give bit-identical results (cf. the reference's transpose-equivalence test,
// tests/test_kernels.cpp:86-116).
__global__ void gemv_omajor(GvParams p) {
  __shared__ double red[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t rblocks = (p.rows + 31) / 32;
  const int64_t items = p.batch * rblocks * p.splits;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int s = static_cast<int>(it % p.splits);
    const int64_t rb = (it / p.splits) % rblocks;
    const int64_t b = it / (p.splits * rblocks);
    int64_t om, ov, oy;
    gv_batch(p, b, om, ov, oy);
    const int64_t o = rb * 32 + tx;
    const int64_t k0 = s * p.chunk, k1 = min(p.K, k0 + p.chunk);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (o < p.rows) {
      const double* mcol = p.M + om + o * p.so;
      const double* vec = p.v + ov;
      for (int64_t kb = k0; kb < k1; kb += 32)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t k = kb + ty + 8 * j;
          if (k < k1) acc[j] = fma(__ldg(mcol + k * p.sk), __ldg(vec + k * p.sv), acc[j]);
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) red[ty + 8 * j][tx] = acc[j];
    __syncthreads();
    if (ty == 0 && o < p.rows) {
      double l[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) l[i] = red[i][tx];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int i = 0; i < off; ++i) l[i] = l[i] + l[i + off];
      gv_store(p, b, o, s, l[0]);
    }
    __syncthreads();
  }
}

__global__ void gemv_finalize(GvParams p) {
  const int64_t n = p.batch * p.rows;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double* part = p.ws + e * p.splits;
    double sum = 0.0;
    for (int s = 0; s < p.splits; ++s) sum += part[s];
    const int64_t o = e % p.rows, b = e / p.rows;
    int64_t om, ov, oy;
    gv_batch(p, b, om, ov, oy);
    double* dst = p.y + oy + gv_row(p, o);
    double r = p.alpha * sum;
    if (p.beta != 0.0) r += p.beta * *dst;
    *dst = r;
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
  // the k-contiguous kernel when rows are not unit-stride (or there is one row)
  const bool kmajor = p.sk == 1 ? (p.so != 1 || p.rows == 1) : (p.so != 1 && p.rows == 1);
  const bool use_k = kmajor || p.rows == 1;
  // The k-chunking depends only on the problem (never on which kernel runs)
  // and chunks are multiples of 32, so the summation order is layout-free.
  int64_t splits = 1;
  {
    const int64_t target = static_cast<int64_t>(sms) * 32;
    const int64_t rows_total = p.batch * p.rows;
    if (rows_total < target)
      splits = std::min<int64_t>((target + rows_total - 1) / rows_total,
                                 std::max<int64_t>(1, d.k / 512));
  }
  splits = std::max<int64_t>(1, std::min<int64_t>(splits, 4096));
  p.chunk = ((d.k + splits - 1) / splits + 31) / 32 * 32;
  splits = (d.k + p.chunk - 1) / p.chunk;
  p.splits = static_cast<int>(splits);
  if (splits > 1) {
    const int64_t need = p.batch * p.rows * splits * 8;
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
    const int64_t warps = p.batch * p.rows * splits;
    const int blocks = static_cast<int>(std::min<int64_t>((warps + 7) / 8, sms * 32LL));
    gemv_kmajor<<<blocks, 256, 0, st.stream>>>(p);
  } else {
    const int64_t items = p.batch * ((p.rows + 31) / 32) * splits;
    const int blocks = static_cast<int>(std::min<int64_t>(items, sms * 16LL));
    gemv_omajor<<<blocks, 256, 0, st.stream>>>(p);
  }
  TCB_LAUNCHED();
  ++launches;
  if (splits > 1) {
    const int64_t n = p.batch * p.rows;
    const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, sms * 8LL));
    gemv_finalize<<<blocks, 256, 0, st.stream>>>(p);
    TCB_LAUNCHED();
    ++launches;
  }
  st.last_info.path = (d.m == 1 && d.n == 1) ? 3 : 2;
  st.last_info.splits = p.splits;
  st.last_info.units = p.batch * p.rows * splits;
  st.last_info.grid = 0;
  st.last_info.launches = launches;
  return TCB_OK;
}

}  // namespace tcb
