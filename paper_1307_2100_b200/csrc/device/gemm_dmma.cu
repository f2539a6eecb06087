// k1/k2 — fp64 GEMM on the B200 DMMA tensor pipe (mma.sync f64 -> SASS
// DMMA.8x8x4), TMA + mbarrier staging, persistent CTAs, deterministic stream-K.
//
// Replaces the reference's ReferenceBackend::gemm (src/kernels_reference.cpp:
// 33-79) *and* the loop-over-GEMM nest around it (src/executor.cpp:119-177):
// one launch evaluates every free-label slice (batch dims) and every
// contracted slice (flattened into K) of a contraction.
//
// Design (sm_100a; fp64 has no tcgen05 kind, so the tensor pipe is reached
// through warp-level mma.sync, fed from shared memory):
//   * CTA tile 128x128x16, 8 consumer warps (2 x 4, warp tile 64x32 = 8x4
//     DMMA 8x8 blocks, 32 independent accumulators/warp) + a producer
//     warpgroup. setmaxnreg hands the producer's registers to the consumers
//     (40 vs 232 per thread): without it a 12-warp CTA caps at 168 registers
//     and the accumulators spill.
//   * smem ring of 32 KB stages with full/empty mbarriers (3 stages next to
//     the 128 KB staging tile, 6 otherwise). One producer thread issues one
//     cp.async.bulk.tensor (TMA, 128B swizzle) per operand per stage through
//     5-D maps built from the operand's index groups — composite M / N / K
//     read in place (recipe L4) — else 128 producer threads issue zero-filling
//     8-byte cp.async arriving on the same mbarrier.
//   * Two smem layouts per operand: "MN-major" (outer index contiguous in
//     global: 8 chunks of 16(outer) x 16(k)) and "K-major" (k contiguous: one
//     16(k) x 128(outer) box); both 128B-swizzled. The k-set of each DMMA
//     k-step is {0,1,4,5}+{0,2,8,10}[j] instead of 4 consecutive k, which makes
//     the fragment loads of *both* layouts exactly 2 wavefronts.
//   * Persistent: grid = min(tiles, #SMs); the producer runs ahead across
//     tile boundaries.
//   * Staged epilogue: consumers drop the accumulators into a swizzled 128 KB
//     staging tile (the smem image of a TMA box of C) and start the next tile;
//     one thread writes the tile with a single TMA tensor store (composite
//     output groups as tensor-map dims), or producer warps 1-3 do plain stores
//     where C has no such map.
//   * Stream-K for small tile grids: CTAs share the (tile, k-block) space from
//     a host-built start table; partial tiles go to a workspace, arrive on a
//     per-tile counter, and every contributor reduces its proportional share
//     in k order (bit-reproducible run to run).
//   * Programmatic dependent launch between consecutive GEMMs on the engine's
//     stream: the next grid's prologue and main loop overlap this one's tail;
//     global writes wait for the previous grid (griddepcontrol).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "tcb_internal.cuh"

namespace tcb {
namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 6;
constexpr int SK_MAX = 160;            // stream-K: most CTAs sharing one launch
constexpr int NCW = 8;                 // consumer (DMMA) warps
constexpr int CTHREADS = NCW * 32;     // 256
constexpr int PTHREADS = 128;          // producer warpgroup
constexpr int NTHREADS = PTHREADS + CTHREADS;
constexpr int STAGE_A = BM * BK * 8;   // 16 KB
constexpr int STAGE_B = BN * BK * 8;   // 16 KB
constexpr int STAGE_BYTES = STAGE_A + STAGE_B;
constexpr int STAGES_STAGED = 3;       // ring depth when the epilogue is staged
constexpr int STAGING_BYTES = BM * BN * 8;  // 128 KB: one accumulator tile
constexpr int TAIL_BYTES = 256 /*barriers*/ + (BM + BN) * 8 /*offset tables*/;
constexpr int SLOT_BYTES = (SK_MAX + 1) * 4;  // stream-K contributor slots (split variant)
constexpr int SMEM_LIMIT = 232448;     // 227 KB opt-in per CTA on sm_100
// Shared-memory layout: [ring][staging (staged epilogue only)][barriers][tables].
template <bool STAGED>
__host__ __device__ constexpr int smem_bytes() {
  return STAGED ? SMEM_LIMIT
                : STAGES * STAGE_BYTES + TAIL_BYTES + SLOT_BYTES + 1024 /*alignment slack*/;
}
static_assert(STAGES_STAGED * STAGE_BYTES + STAGING_BYTES + TAIL_BYTES + 512 <= SMEM_LIMIT,
              "staged layout must fit with alignment slack");

// How the producer derives the 5 coordinates of an operand tensor map from
// the (outer index, k index, batch index) of a tile origin: dimension d reads
// source src[d] (0 outer, 1 k, 2 batch, 3 constant 0) and takes
// (value / div[d]) % mod[d] (mod 0: no modulus). Composite index groups —
// several tensor dimensions forming one GEMM index — are thereby read in
// place, with no permutation pass. Outer and batch coordinates are computed
// once per work unit, k coordinates once per stage. nbox: 1 when one box
// covers the operand's whole stage; 8 for MN-major operands whose outer
// extent is not a multiple of 16 (eight 16x16 boxes, dimension 0 advancing
// by 16).
struct MapProg {
  unsigned div[5], mod[5];
  int src[5];
  int nbox;
  int kdim;   // the single k dim when k is not composite (coordinate = k), else -1
};

struct Params {
  const double* A;
  const double* B;
  double* C;
  int64_t M, N, K;
  int64_t a_so, a_sk, b_so, b_sk;  // operand strides along (outer, k)
  int c_nrow, c_ncol;
  int64_t c_row_ext[TCB_MAX_DIMS], c_row_str[TCB_MAX_DIMS];
  int64_t c_col_ext[TCB_MAX_DIMS], c_col_str[TCB_MAX_DIMS];
  int nbatch;
  int64_t bat_ext[TCB_MAX_DIMS], bat_sa[TCB_MAX_DIMS], bat_sb[TCB_MAX_DIMS], bat_sc[TCB_MAX_DIMS];
  double alpha, beta;
  int alpha_ne1, beta_nz;  // alpha != 1, beta != 0 (decided on the host)
  int tiles_m, tiles_n, splits, kblocks;
  int64_t units;                // tiles (data-parallel work items)
  // stream-K (split variant): tiles [0, dp_tiles) go whole, round robin
  // (data-parallel phase); then CTA c owns k-blocks [sk_start[c],
  // sk_start[c+1]) of the flattened (tile, k-block) space (absolute
  // positions, from dp_tiles * kblocks on); sk_grid CTAs
  int sk_grid;
  int dp_tiles;
  int64_t work;
  int sk_start[SK_MAX + 1];
  double* ws;
  unsigned* counters;
  unsigned epoch;  // split-K: counters reach (epoch+1)*splits in this launch
  unsigned long long* trace;  // TCB_TRACE diagnostics: per-CTA phase timestamps (or null)
  int diag;                   // TCB_DIAG bits (diagnostics only): 1 = storers skip C writes
  // TMA coordinate programs of the A and B tensor maps (see MapProg)
  MapProg pa, pb;
  // staged epilogue: C written by one TMA tensor store per tile (c_tma) with
  // coordinate program pc (sources: 0 m origin, 1 n origin, 2 batch)
  int c_tma;
  int c_red;                  // beta == 1: the TMA store is a reduce-add into C
  MapProg pc;
  // tile raster: groups of `raster_g` m-tiles per n sweep (raster_n = 0), or
  // of raster_g n-tiles per m sweep (raster_n = 1, keeps that set of B panels
  // resident in L2 while A streams)
  int raster_g, raster_n;
  // k-pacing (long-k launches): the producers of all CTAs announce every
  // 2^pace_shift issued k-blocks on one global counter and do not start
  // epoch e before every CTA has announced epoch e - pace_slack, so the CTAs
  // that share an operand panel stay within a few epochs of each other and
  // its k-slices are fetched from DRAM once, then hit in L2. The counter is
  // monotonic across launches: this launch's announcements start at
  // pace_base and total pace_total per CTA. A performance hint only: a wait
  // gives up after a timeout, so it never blocks progress.
  unsigned long long* pace;
  unsigned long long pace_base;
  int pace_shift, pace_slack, pace_grid;
  unsigned pace_total;
  // gate (tcb_gemm_gated): the producer issues no operand load before
  // *gate >= gate_value — a device-side dependency on an upload stream
  // (tcb_stream_write_value), so consecutive GEMMs keep programmatic
  // dependent launch instead of a host-visible stream wait between them
  const unsigned long long* gate;
  unsigned long long gate_value;
  // whole tiles of odd waves issue their k-blocks in descending order: the
  // k-slices a wave used last are the next wave's first, still in L2 (the
  // consumers are order-agnostic; the tile's sum order is fixed per tile)
  int kflip;
  // L2 eviction priority of the operand loads (0 = default, 1 = evict_first,
  // 2 = evict_last): the raster's resident panel group evict_last, the
  // streamed operand evict_first, so the stream does not push the group out
  int a_hint, b_hint, c_hint;
  // prefetch each whole tile's C into L2 ahead of its epilogue (beta != 0
  // with a register-path epilogue; plain column-major C, no batch)
  int c_pf;
};

// Params + three tensor maps are the kernel's parameters: stay within the
// classic 4 KB (a 6 KB block carrying per-CTA tables indexed at run time
// failed a batched stream-K launch; not root-caused, so not repeated)
static_assert(sizeof(Params) + 3 * sizeof(CUtensorMap) <= 4096, "kernel parameters above 4 KB");

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const double* src, bool valid) {
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void tma_load5(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                          int c0, int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
      : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void tma_load5_hint(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                               int c0, int c1, int c2, int c3, int c4,
                                               uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar),
      "l"(pol)
      : "memory");
}
// L2 policies: 1 = evict_first (streamed operand), 2 = evict_last (resident set)
__device__ __forceinline__ uint64_t l2_policy(int hint) {
  uint64_t pol;
  if (hint == 1)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_store5(const CUtensorMap* map, uint32_t src, int c0, int c1,
                                           int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group"
      " [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(src)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// C += tile: the TMA engine adds the staged tile to C in L2 (one f64 add per
// element, so fma(1, C, v) exactly) — beta == 1 without a single C load by the SM
__device__ __forceinline__ void tma_reduce_add5(const CUtensorMap* map, uint32_t src, int c0,
                                                int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.5d.global.shared::cta.add.tile.bulk_group"
      " [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(src)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store5_hint(const CUtensorMap* map, uint32_t src, int c0,
                                                int c1, int c2, int c3, int c4, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group.L2::cache_hint"
      " [%0, {%1, %2, %3, %4, %5}], [%6], %7;" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(src), "l"(pol)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// Programmatic dependent launch: let the next grid in the stream start (its
// CTAs are scheduled as ours exit), and wait for the previous grid to have
// completed before this thread's first global write.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// the bulk stores have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// all bulk stores are complete (visible in global memory)
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// order this thread's generic-proxy shared-memory writes before async-proxy reads
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Byte offset of accumulator (m, n) of a tile in the staging buffer: 8 boxes
// (m / 16) of [n 128][m 16] with the 128-byte swizzle — the smem image of
// the output tensor map's box, conflict-free for the consumers' fragment
// stores and for the fallback storers' column reads.
__device__ __forceinline__ uint32_t stage_off(int m, int n) {
  return (m >> 4) * 16384 + n * 128 + (((((m & 15) >> 1) ^ (n & 7))) << 4) + ((m & 1) << 3);
}
// Diagnostics (TCB_TRACE): %globaltimer at phase boundaries, first unit only.
__device__ __forceinline__ void trace_mark(const Params& p, int slot, bool leader) {
  if (p.trace != nullptr && leader) {
    unsigned long long t;
    if (p.diag & 32)  // TCB_DIAG bit 32: SM clock cycles instead of ns
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    else
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[blockIdx.x * 32 + slot] = t;
  }
}
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(CTHREADS) : "memory");
}
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// ------------------------------------------------------------ smem layouts
// Byte offset of element (o = outer index in [0,128), k in [0,16)) in a stage.
template <bool KMAJOR>
__device__ __forceinline__ uint32_t tile_off(int o, int k) {
  if (KMAJOR)  // one 16(k) x 128(o) box: row = o (128 B), chunk = k/2 ^ (o%8)
    return o * 128 + ((((k >> 1) ^ (o & 7))) << 4) + ((k & 1) << 3);
  // 8 boxes of 16(o) x 16(k): box o/16, row = k (128 B), chunk = (o%16)/2 ^ (k%8)
  return (o >> 4) * 2048 + k * 128 + (((((o & 15) >> 1) ^ (k & 7))) << 4) + ((o & 1) << 3);
}

// k index of lane-quad q in k-step j of a 16-wide k block (see header note).
__device__ __forceinline__ constexpr int kstep_k(int j, int q) {
  return (q & 1) | ((q >> 1) << 2) | ((j & 1) << 1) | ((j >> 1) << 3);
}

// One k-block of a consumer warp: 4 k-steps of 12 fragment loads + 32 DMMA.
// EPI != 0 (the last k-block of a segment): the last k-step's DMMAs are
// interleaved with the accumulators' stores, LAG DMMAs behind the one that
// finishes each accumulator, so the tensor pipe keeps issuing while the tile
// leaves the registers — EPI 1: into the staging tile of the staged epilogue
// (a separate store pass idles the pipe for ~0.4 us per tile: 128 KB at the
// shared-memory store rate); EPI 2: a stream-K partial into its workspace
// slot (`part`: this thread's first pair, pairs CTHREADS apart).
template <bool A_KMAJOR, bool B_KMAJOR, int EPI>
__device__ __forceinline__ void consume_kblock(double (&acc)[8][4][2], uint32_t sA, uint32_t sB,
                                               const uint32_t (&offA)[4],
                                               const uint32_t (&offB)[4], int wm, int wn,
                                               uint32_t stg, double2* part, int r, int q) {
  constexpr int LAG = 6;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double a[8], b[4];
#pragma unroll
    for (int im = 0; im < 8; ++im) {
      const uint32_t addr = A_KMAJOR ? sA + (wm * 64 + im * 8) * 128 + offA[j]
                                     : sA + (wm * 4 + (im >> 1)) * 2048 + (j >> 1) * 1024 +
                                           offA[(j & 1) | ((im & 1) << 1)];
      a[im] = lds64(addr);
    }
#pragma unroll
    for (int in = 0; in < 4; ++in) {
      const uint32_t addr = B_KMAJOR ? sB + (wn * 32 + in * 8) * 128 + offB[j]
                                     : sB + (wn * 2 + (in >> 1)) * 2048 + (j >> 1) * 1024 +
                                           offB[(j & 1) | ((in & 1) << 1)];
      b[in] = lds64(addr);
    }
    if (EPI != 0 && j == 3) {
#pragma unroll
      for (int v = 0; v < 32 + LAG; ++v) {
        if (v < 32) dmma(acc[v >> 2][v & 3], a[v >> 2], b[v & 3]);
        if (v >= LAG) {
          const int im = (v - LAG) >> 2, in = (v - LAG) & 3;
          if (EPI == 2) {
            asm volatile("st.global.cg.v2.f64 [%0], {%1, %2};" ::"l"(part + (im * 4 + in) * CTHREADS),
                         "d"(acc[im][in][0]), "d"(acc[im][in][1])
                         : "memory");
          } else {
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              const uint32_t ad =
                  stg + stage_off(wm * 64 + im * 8 + r, wn * 32 + in * 8 + 2 * q + jj);
              asm volatile("st.shared.f64 [%0], %1;" ::"r"(ad), "d"(acc[im][in][jj]) : "memory");
            }
          }
        }
      }
    } else {
#pragma unroll
      for (int im = 0; im < 8; ++im)
#pragma unroll
        for (int in = 0; in < 4; ++in) dmma(acc[im][in], a[im], b[in]);
    }
  }
}

// ------------------------------------------------------------- unit decode
// Index arithmetic below is 32-bit unsigned: the host guarantees units,
// batch count, M and N (and every group extent) are < 2^31, so no 64-bit
// division routine is ever called from the kernel.
struct Unit {
  unsigned batch;
  int tm, tn, split;
};

__device__ __forceinline__ Unit decode_unit(const Params& p, int64_t tile) {
  const unsigned t = static_cast<unsigned>(tile);
  Unit r;
  r.split = 0;
  const unsigned per_batch = static_cast<unsigned>(p.tiles_m) * static_cast<unsigned>(p.tiles_n);
  r.batch = t / per_batch;
  const unsigned tt = t - r.batch * per_batch;
  // grouped raster: raster_g m-tiles share each n-tile sweep (L2 reuse of B
  // panels across the group), or with raster_n raster_g n-tiles share each
  // m-tile sweep (a resident set of B panels while A streams through)
  const int G = p.raster_g;
  const int lead = p.raster_n ? p.tiles_n : p.tiles_m;
  const unsigned cross = static_cast<unsigned>(p.raster_n ? p.tiles_m : p.tiles_n);
  const unsigned group_span = static_cast<unsigned>(G) * cross;
  const unsigned g = tt / group_span;
  const int first = static_cast<int>(g * static_cast<unsigned>(G));
  const unsigned gsize = static_cast<unsigned>(min(G, lead - first));
  const unsigned w = tt - g * group_span;
  const int a = first + static_cast<int>(w % gsize), b = static_cast<int>(w / gsize);
  r.tm = p.raster_n ? b : a;
  r.tn = p.raster_n ? a : b;
  return r;
}

__device__ __forceinline__ void batch_offsets(const Params& p, unsigned b, int64_t& oa,
                                              int64_t& ob, int64_t& oc, int* coords) {
  oa = ob = oc = 0;
  for (int i = 0; i < p.nbatch; ++i) {
    const unsigned e = static_cast<unsigned>(p.bat_ext[i]);
    const unsigned nb = b / e;
    const unsigned c = b - nb * e;
    b = nb;
    coords[i] = static_cast<int>(c);
    oa += static_cast<int64_t>(c) * p.bat_sa[i];
    ob += static_cast<int64_t>(c) * p.bat_sb[i];
    oc += static_cast<int64_t>(c) * p.bat_sc[i];
  }
}

__device__ __forceinline__ int64_t composite(int64_t idx64, int n, const int64_t* ext,
                                             const int64_t* str) {
  unsigned idx = static_cast<unsigned>(idx64);
  int64_t off = 0;
  for (int i = 0; i < n - 1; ++i) {
    const unsigned e = static_cast<unsigned>(ext[i]);
    const unsigned q = idx / e;
    off += static_cast<int64_t>(idx - q * e) * str[i];
    idx = q;
  }
  return off + static_cast<int64_t>(idx) * str[n - 1];
}

// Outer and batch coordinates of a tile origin (k dims: 0).
__device__ __forceinline__ void unit_coords(const MapProg& g, unsigned o, unsigned b,
                                            int (&c)[5]) {
#pragma unroll
  for (int d = 0; d < 5; ++d) {
    const int s = g.src[d];
    if (g.src[d] == 0 || g.src[d] == 2) {
      unsigned v = s == 0 ? o : b;
      if (g.div[d] != 1u) v /= g.div[d];
      if (g.mod[d] != 0u) v %= g.mod[d];
      c[d] = static_cast<int>(v);
    } else {
      c[d] = 0;
    }
  }
}

// ------------------------------------------------------------------ kernel
// The work of one CTA as segments (tile, k-blocks [kb0, kb1)):
//   * data-parallel: whole tiles u = blockIdx.x, blockIdx.x + gridDim.x, ...;
//   * stream-K (split variant, tiles < SMs): the CTA's contiguous share
//     [sk_start[c], sk_start[c+1]) of the flattened (tile, k-block) space —
//     at most two segments (shares are shorter than a tile's k-blocks).
template <bool SK>
struct SegIter {
  int64_t u;         // data-parallel: tile index
  int64_t pos, end;  // stream-K: position in the (tile, k-block) space
  __device__ __forceinline__ void init(const Params& p) {
    u = blockIdx.x;
    if (SK) {
      pos = p.sk_start[blockIdx.x];
      end = p.sk_start[blockIdx.x + 1];
    }
  }
  __device__ __forceinline__ bool next(const Params& p, int64_t& tile, int& kb0, int& kb1) {
    if (SK) {
      if (u < p.dp_tiles) {  // data-parallel phase: whole tiles
        tile = u;
        kb0 = 0;
        kb1 = p.kblocks;
        u += gridDim.x;
        return true;
      }
      if (pos >= end) return false;
      tile = pos / p.kblocks;
      kb0 = static_cast<int>(pos - tile * p.kblocks);
      kb1 = static_cast<int>(min(static_cast<int64_t>(p.kblocks), kb0 + (end - pos)));
      pos = tile * p.kblocks + kb1;
      return true;
    }
    if (u >= p.units) return false;
    tile = u;
    kb0 = 0;
    kb1 = p.kblocks;
    u += gridDim.x;
    return true;
  }
};

// stream-K: the CTA whose share holds position pos — the last c with
// sk_start[c] <= pos. Shares are near-equal, so a proportional guess corrected
// by a step or two replaces a binary search (8 dependent parameter loads).
__device__ __forceinline__ int sk_owner(const Params& p, int pos) {
  const int n = p.sk_grid, base = p.sk_start[0];
  const float span = static_cast<float>(p.sk_start[n] - base);
  int c = span > 0.f ? static_cast<int>(static_cast<float>(pos - base) * n / span) : 0;
  c = min(max(c, 0), n - 1);
  while (c > 0 && p.sk_start[c] > pos) --c;
  while (c + 1 < n && p.sk_start[c + 1] <= pos) ++c;
  return c;
}

// Stream-K reduction assignment: whether CTA b sums part of tile t's pairs,
// and which ([p0, p1) of `pairs`). Each contributor reduces in one tile
// only — its only tile, or, when its share crosses a tile boundary, the one
// it computed more of (the later one on a tie) — with a pair range in
// proportion to its whole share; a tile that no contributor prefers is
// reduced whole by its largest contributor. (When crossing CTAs also
// reduced a slice of their second tile they waited for two tiles' partials
// and ended the launch 3-4 us after the others on cfg1.) Computed the same
// way by every thread from the share table: no per-launch table in Params.
__device__ __forceinline__ bool sk_reduce_range(const Params& p, int b, int t, int pairs, int& p0,
                                                int& p1, int& first, int& last) {
  // 32-bit positions (the host keeps tiles * kblocks < 2^31); O(1): only the
  // tile's first and last contributors can cross into a neighbour tile
  const int kb = p.kblocks, t0k = t * kb, t1k = t0k + kb;
  first = sk_owner(p, t0k);
  last = sk_owner(p, t1k - 1);
  if (first == last) return false;  // one contributor: it stored the whole tile itself
  const int fa = p.sk_start[first], fe = p.sk_start[first + 1];
  const int la = p.sk_start[last], le = p.sk_start[last + 1];
  // first prefers t unless it computed more of t-1; last prefers t unless it
  // computed at least as much of t+1 (ties go to the later tile)
  const bool f_pref = fa == t0k || t0k - fa <= fe - t0k;
  const bool l_pref = le <= t1k || t1k - la > le - t1k;
  const int F = f_pref ? fe - fa : 0;
  const int L = l_pref ? le - la : 0;
  const int M = la - p.sk_start[first + 1];  // the contributors strictly inside t
  const int W = F + M + L;
  if (W == 0) {  // no contributor prefers t: the larger of the two sums it all
    const int best = (fe - t0k) >= (t1k - la) ? first : last;
    if (b != best) return false;
    p0 = 0;
    p1 = pairs;
    return true;
  }
  int before, mine;
  if (b == first) {
    before = 0;
    mine = F;
  } else if (b == last) {
    before = F + M;
    mine = L;
  } else if (b > first && b < last) {
    before = F + p.sk_start[b] - p.sk_start[first + 1];
    mine = p.sk_start[b + 1] - p.sk_start[b];
  } else {
    return false;
  }
  if (mine == 0) return false;
  p0 = static_cast<int>(static_cast<int64_t>(pairs) * before / W);
  p1 = static_cast<int>(static_cast<int64_t>(pairs) * (before + mine) / W);
  return true;
}

// Wait for the gate (see Params), then order the async-proxy (TMA) operand
// reads after the acquire.
__device__ __forceinline__ void gate_wait(const Params& p) {
  unsigned long long v;
  const unsigned long long t0 = wait_clock_ns();
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p.gate) : "memory");
    if (v >= p.gate_value) break;
    __nanosleep(256);
    if (wait_clock_ns() - t0 > kWaitTrapNs) __trap();  // the gate was never opened
  }
  asm volatile("fence.proxy.async;" ::: "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// k-pacing (see Params): announce that epoch e - 1 is issued, then wait (at
// most ~40 us; after a timeout the CTA stops waiting for the rest of the
// launch) until every CTA has announced epoch e - pace_slack.
__device__ __forceinline__ void pace_epoch(const Params& p, uint32_t e, bool& wait_ok) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(p.pace) : "memory");
  if (!wait_ok || e < static_cast<uint32_t>(p.pace_slack)) return;
  const unsigned long long target =
      p.pace_base + static_cast<unsigned long long>(e - p.pace_slack + 1) * p.pace_grid;
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p.pace) : "memory");
  if (v >= target) return;
  const unsigned long long t0 = global_ns();
  do {
    __nanosleep(128);
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p.pace) : "memory");
    if (global_ns() - t0 > 40000) {
      wait_ok = false;
      return;
    }
  } while (v < target);
}

// Producer-side iterator over this CTA's (segment, k-block) sequence. All
// per-segment address math happens once per segment here, in the producer
// warpgroup, never on the consumer warps.
template <bool SK>
struct LoadIter {
  SegIter<SK> it;
  int kb, kb1;
  int m0, n0;            // tile origin (TMA coordinates are int32)
  int64_t oa, ob;        // batch offsets (cp.async path)
  int ca[5], cb[5];      // TMA: outer + batch coordinates of the segment's tile
  int mirror;            // >= 0: k-blocks issued as mirror - kb (descending)
  bool valid;
  bool whole;            // the segment is a whole tile

  template <bool USE_TMA>
  __device__ __forceinline__ void start(const Params& p) {
    it.init(p);
    start_seg<USE_TMA>(p);
  }
  template <bool USE_TMA>
  __device__ __forceinline__ void start_seg(const Params& p) {
    int64_t tile;
    valid = it.next(p, tile, kb, kb1);
    if (!valid) return;
    whole = kb == 0 && kb1 == p.kblocks;
    mirror = (p.kflip && kb == 0 && kb1 == p.kblocks &&
              ((static_cast<unsigned>(tile) / gridDim.x) & 1u))
                 ? kb1 - 1
                 : -1;
    const Unit un = decode_unit(p, tile);
    m0 = un.tm * BM;
    n0 = un.tn * BN;
    if (USE_TMA) {
      unit_coords(p.pa, static_cast<unsigned>(m0), un.batch, ca);
      unit_coords(p.pb, static_cast<unsigned>(n0), un.batch, cb);
    } else {
      int bc[TCB_MAX_DIMS];
      int64_t oc;
      batch_offsets(p, un.batch, oa, ob, oc, bc);
    }
  }
  template <bool USE_TMA>
  __device__ __forceinline__ void advance(const Params& p) {
    if (++kb == kb1) start_seg<USE_TMA>(p);
  }
};

__device__ __forceinline__ unsigned prog_coord(const MapProg& g, int d, unsigned v) {
  if (g.div[d] != 1u) v /= g.div[d];
  if (g.mod[d] != 0u) v %= g.mod[d];
  return v;
}
// k coordinate of dimension d at k index k0 (0 for outer / batch dims)
__device__ __forceinline__ int k_coord(const MapProg& g, int d, unsigned k0) {
  return g.src[d] == 1 ? static_cast<int>(prog_coord(g, d, k0)) : 0;
}

// Issue one k-block of both operands into a stage. TMA: one thread, 5-D maps
// (lead, other, 3 batch dims). cp.async: the 128 producer threads.
template <bool A_KMAJOR, bool B_KMAJOR, bool USE_TMA, typename Iter>
__device__ __forceinline__ void issue_stage(const Params& p, const CUtensorMap& tmA,
                                            const CUtensorMap& tmB, const Iter& li,
                                            uint32_t sA, uint32_t full, int ptid) {
  const int k0 = (li.mirror >= 0 ? li.mirror - li.kb : li.kb) * BK;
  const uint32_t sB = sA + STAGE_A;
  if (USE_TMA) {
    mbar_expect_tx(full, STAGE_BYTES);
    const unsigned k0u = static_cast<unsigned>(k0);
    {
      int c[5];
      if (p.pa.kdim >= 0) {
#pragma unroll
        for (int d = 0; d < 5; ++d) c[d] = li.ca[d] + (d == p.pa.kdim ? k0 : 0);
      } else {
#pragma unroll
        for (int d = 0; d < 5; ++d) c[d] = li.ca[d] + k_coord(p.pa, d, k0u);
      }
      if (p.a_hint) {
        const uint64_t pol = l2_policy(p.a_hint);
#pragma unroll 1
        for (int i = 0; i < p.pa.nbox; ++i, c[0] += 16)
          tma_load5_hint(sA + i * 2048, &tmA, full, c[0], c[1], c[2], c[3], c[4], pol);
      } else {
#pragma unroll 1
        for (int i = 0; i < p.pa.nbox; ++i, c[0] += 16)
          tma_load5(sA + i * 2048, &tmA, full, c[0], c[1], c[2], c[3], c[4]);
      }
    }
    {
      int c[5];
      if (p.pb.kdim >= 0) {
#pragma unroll
        for (int d = 0; d < 5; ++d) c[d] = li.cb[d] + (d == p.pb.kdim ? k0 : 0);
      } else {
#pragma unroll
        for (int d = 0; d < 5; ++d) c[d] = li.cb[d] + k_coord(p.pb, d, k0u);
      }
      if (p.b_hint) {
        const uint64_t pol = l2_policy(p.b_hint);
#pragma unroll 1
        for (int i = 0; i < p.pb.nbox; ++i, c[0] += 16)
          tma_load5_hint(sB + i * 2048, &tmB, full, c[0], c[1], c[2], c[3], c[4], pol);
      } else {
#pragma unroll 1
        for (int i = 0; i < p.pb.nbox; ++i, c[0] += 16)
          tma_load5(sB + i * 2048, &tmB, full, c[0], c[1], c[2], c[3], c[4]);
      }
    }
  } else {
    const double* Ab = p.A + li.oa;
    const double* Bb = p.B + li.ob;
    // 2048 elements per operand tile, 16 per producer thread; the thread order
    // follows the operand's unit-stride index so warps read contiguous memory.
#pragma unroll 4
    for (int i = 0; i < (BM * BK) / PTHREADS; ++i) {
      const int idx = ptid + PTHREADS * i;
      const int o = (p.a_so == 1) ? (idx & (BM - 1)) : (idx >> 4);
      const int k = (p.a_so == 1) ? (idx >> 7) : (idx & 15);
      const int64_t gm = li.m0 + o, gk = k0 + k;
      const bool ok = gm < p.M && gk < p.K;
      cp_async8(sA + tile_off<A_KMAJOR>(o, k), ok ? Ab + gm * p.a_so + gk * p.a_sk : p.A, ok);
    }
#pragma unroll 4
    for (int i = 0; i < (BN * BK) / PTHREADS; ++i) {
      const int idx = ptid + PTHREADS * i;
      const int o = (p.b_so == 1) ? (idx & (BN - 1)) : (idx >> 4);
      const int k = (p.b_so == 1) ? (idx >> 7) : (idx & 15);
      const int64_t gn = li.n0 + o, gk = k0 + k;
      const bool ok = gn < p.N && gk < p.K;
      cp_async8(sB + tile_off<B_KMAJOR>(o, k), ok ? Bb + gn * p.b_so + gk * p.b_sk : p.B, ok);
    }
    cp_async_arrive_noinc(full);
  }
}

// Epilogue: thread's 8x4x2 accumulators -> C through the tile's offset tables.
// BETA: the old C values of two accumulator rows (16 loads) are fetched
// before any of their stores. Written element by element (load, DFMA, store)
// the compiler must keep every load behind the previous store (the pointers
// may alias for all it knows), which serialises 64 L2 round trips per tile:
// ~22 us per 128 x 128 tile, 0.5 % of a cfg5 K-slab GEMM (SASS: LDG, DFMA,
// STG chains; measured 122.4 vs 121.8 ms for a 64-l slab with beta = 1 / 0).
template <bool BETA>
__device__ __forceinline__ void store_tile(const double (&acc)[8][4][2], double* Cb,
                                           const int64_t* s_row, const int64_t (&coff)[4][2],
                                           const bool (&cok)[4][2], int wm, int r, double alpha,
                                           double beta) {
  constexpr int G = 2;  // accumulator rows per batch of old-C loads
#pragma unroll
  for (int im0 = 0; im0 < 8; im0 += G) {
    double* row[G];
    bool rok[G];
    double old[G][4][2];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int64_t roff = s_row[wm * 64 + (im0 + g) * 8 + r];
      row[g] = Cb + roff;
      rok[g] = roff >= 0;
    }
    if (BETA) {
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int in = 0; in < 4; ++in)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
            old[g][in][jj] = (rok[g] && cok[in][jj]) ? *(row[g] + coff[in][jj]) : 0.0;
    }
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int in = 0; in < 4; ++in)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          double v = alpha * acc[im0 + g][in][jj];
          if (BETA) v = fma(beta, old[g][in][jj], v);
          if (rok[g] && cok[in][jj]) *(row[g] + coff[in][jj]) = v;
        }
  }
}

// Stream-K fix-up: sum pairs [p0, p1) of a tile over its S contributors'
// workspace slots in contributor (= k) order and write them to C.
// Each thread owns up to RED pairs per pass and issues the partial loads of CB
// contributors before summing.
constexpr int SK_RED_CB = 10;
template <int CB>
__device__ __forceinline__ void sk_reduce_pairs(const Params& p, const double2* ws,
                                                const int* s_slot, const int64_t* s_row,
                                                const int64_t* s_col, double* Cb, int S, int p0,
                                                int p1, int ctid, bool use_beta) {
  constexpr int PAIRS = BM * BN / 2;
  constexpr int RED = 4;  // 2: -2 %, 8: -0.6 % on cfg1 (measured)
#pragma unroll 1
  for (int pb = p0 + ctid; pb < p1; pb += CTHREADS * RED) {
    double2 sum[RED];
#pragma unroll
    for (int i = 0; i < RED; ++i) sum[i] = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int sp0 = 0; sp0 < S; sp0 += CB) {
      double2 v[CB][RED];
#pragma unroll
      for (int jj = 0; jj < CB; ++jj) {
        const int64_t base = sp0 + jj < S ? static_cast<int64_t>(s_slot[sp0 + jj]) * PAIRS : 0;
#pragma unroll
        for (int i = 0; i < RED; ++i) {
          const int pi = pb + i * CTHREADS;
          v[jj][i] = (sp0 + jj < S && pi < p1) ? __ldcg(ws + base + pi) : make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int jj = 0; jj < CB; ++jj)
#pragma unroll
        for (int i = 0; i < RED; ++i)
          if (sp0 + jj < S) {  // contributor order 0..S-1
            sum[i].x += v[jj][i].x;
            sum[i].y += v[jj][i].y;
          }
    }
#pragma unroll
    for (int i = 0; i < RED; ++i) {
      const int pi = pb + i * CTHREADS;
      if (pi >= p1) continue;
      // pair index -> (m, n): v = pi / 256 (im = v/4, in = v%4), thread t = pi % 256
      const int v = pi >> 8, tt = pi & 255;
      const int tw = tt >> 5, tl2 = tt & 31;
      const int m = (tw & 1) * 64 + (v >> 2) * 8 + (tl2 >> 2);
      const int n = (tw >> 1) * 32 + (v & 3) * 8 + 2 * (tl2 & 3);
      const int64_t roff = s_row[m];
      if (roff < 0) continue;
      const double sv[2] = {sum[i].x, sum[i].y};
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int64_t coff = s_col[n + jj];
        if (coff < 0) continue;
        double* dst = Cb + roff + coff;
        double vv = p.alpha * sv[jj];
        if (use_beta) vv += p.beta * *dst;
        *dst = vv;
      }
    }
  }
}

// 384 threads: warpgroup 0 = producer (TMA: one elected thread; cp.async: all
// 128), warpgroups 1-2 = 8 DMMA consumer warps. setmaxnreg moves registers
// from the producer (40/thread) to the consumers (232/thread) so the 64-double
// accumulator tile never spills (a plain 9- or 12-warp CTA caps at 168).
template <bool A_KMAJOR, bool B_KMAJOR, bool USE_TMA, bool SPLITK>
__global__ void __launch_bounds__(NTHREADS, 1)
    dgemm_dmma_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmC) {
  // Staged epilogue (TMA, no split-K): consumers dump the accumulator tile into
  // shared memory and go straight on to the next tile's main loop; producer
  // warps 1-3 apply alpha/beta and write C from there, overlapped with DMMA.
  constexpr bool STAGED = USE_TMA && !SPLITK;
  constexpr int NST = STAGED ? STAGES_STAGED : STAGES;
  extern __shared__ unsigned char smem_raw[];
  // 1024-aligned base (128B-swizzled TMA boxes) computed in the 32-bit shared
  // window: the main loop's barrier / stage addresses then rematerialise from
  // constants instead of re-deriving a generic pointer (S2R of the shared
  // window) every k-block
  const uint32_t raw = smem_u32(smem_raw);
  uint32_t s_base = (raw + 1023u) & ~1023u;
  asm volatile("mov.b32 %0, %0;" : "+r"(s_base));  // opaque: kept in a register
  unsigned char* smem = smem_raw + (s_base - raw);
  double* staging = reinterpret_cast<double*>(smem + NST * STAGE_BYTES);
  unsigned char* tail = smem + NST * STAGE_BYTES + (STAGED ? STAGING_BYTES : 0);
  const uint32_t tail_u32 = s_base + NST * STAGE_BYTES + (STAGED ? STAGING_BYTES : 0);
  const uint32_t full0 = tail_u32;                 // full[s]  = full0 + 8s
  const uint32_t empty0 = tail_u32 + 8 * NST;      // empty[s] = empty0 + 8s
  const uint32_t stg_full = tail_u32 + 16 * NST;   // staging holds a tile
  const uint32_t stg_empty = stg_full + 8;         // staging drained
  // per-tile output offsets: composite row(m) / col(n) of the tile, -1 = outside C
  int64_t* s_row = reinterpret_cast<int64_t*>(tail + 256);
  int64_t* s_col = s_row + BM;
  int* s_slot = reinterpret_cast<int*>(s_col + BN);  // stream-K contributor slots

  const int tid = threadIdx.x;
  if (tid == 0) {
    if (tail + TAIL_BYTES + (STAGED ? 0 : SLOT_BYTES) > smem_raw + smem_bytes<STAGED>()) __trap();
    for (int s = 0; s < NST; ++s) {
      mbar_init(full0 + 8 * s, USE_TMA ? 1 : PTHREADS);
      mbar_init(empty0 + 8 * s, NCW);
    }
    mbar_init(stg_full, CTHREADS);
    mbar_init(stg_empty, p.c_tma ? 1 : PTHREADS - 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (USE_TMA) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      if (STAGED && p.c_tma)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmC)) : "memory");
    }
  }
  __syncthreads();
  pdl_launch_dependents();

  if (tid < PTHREADS) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;" ::: "memory");
    if (STAGED && tid >= 32) {
      // ========================== storers (warps 1-3) ==========================
      const int stid = tid - 32;  // 0..95
      const int swarp = stid >> 5, slane = stid & 31;
      uint32_t t = 0;
      if (p.c_tma) {
        // one thread: a TMA tensor store per tile straight from the staging
        // buffer (no register traffic, clipped at the C edges)
        if (stid != 0) return;
        const uint32_t stg = smem_u32(staging);
#pragma unroll 1
        for (int64_t u = blockIdx.x; u < p.units; u += gridDim.x, ++t) {
          const Unit un = decode_unit(p, u);
          int c[5];
#pragma unroll
          for (int d = 0; d < 5; ++d) {
            const int src = p.pc.src[d];
            unsigned v = src == 0 ? static_cast<unsigned>(un.tm * BM)
                                  : (src == 1 ? static_cast<unsigned>(un.tn * BN)
                                              : (src == 2 ? un.batch : 0u));
            c[d] = static_cast<int>(prog_coord(p.pc, d, v));
          }
          mbar_wait(stg_full, t & 1);
          pdl_wait();
          if (p.c_red)
            tma_reduce_add5(&tmC, stg, c[0], c[1], c[2], c[3], c[4]);
          else if (p.c_hint)
            tma_store5_hint(&tmC, stg, c[0], c[1], c[2], c[3], c[4], l2_policy(p.c_hint));
          else if (!(p.diag & 16))  // TCB_DIAG bit 16: no C store (timing experiment)
            tma_store5(&tmC, stg, c[0], c[1], c[2], c[3], c[4]);
          bulk_wait_read();  // staging may be overwritten once read
          mbar_arrive(stg_empty);
        }
        bulk_wait_all();
        return;
      }
#pragma unroll 1
      for (int64_t u = blockIdx.x; u < p.units; u += gridDim.x, ++t) {
        const Unit un = decode_unit(p, u);
        int bc[TCB_MAX_DIMS];
        int64_t oa, ob, oc;
        batch_offsets(p, un.batch, oa, ob, oc, bc);
        asm volatile("bar.sync 2, 96;" ::: "memory");  // previous tile's tables consumed
        for (int i = stid; i < BM + BN; i += 96) {
          if (i < BM) {
            const int64_t m = static_cast<int64_t>(un.tm) * BM + i;
            s_row[i] = m < p.M ? composite(m, p.c_nrow, p.c_row_ext, p.c_row_str) : -1;
          } else {
            const int64_t n = static_cast<int64_t>(un.tn) * BN + (i - BM);
            s_col[i - BM] = n < p.N ? composite(n, p.c_ncol, p.c_col_ext, p.c_col_str) : -1;
          }
        }
        asm volatile("bar.sync 2, 96;" ::: "memory");
        mbar_wait(stg_full, t & 1);
        pdl_wait();
        double* Cb = p.C + oc;
        // warp w writes columns n = w, w+3, ...; lanes walk m (coalesced in C).
        // alpha was applied by the consumers; plain copies keep the FP64 pipe
        // (shared with DMMA) free unless beta needs a DFMA.
        const bool use_beta = p.beta_nz != 0;  // host-side flag: no FP64 compare here
        int64_t roff[BM / 32];
#pragma unroll
        for (int j = 0; j < BM / 32; ++j) roff[j] = s_row[slane + 32 * j];
        if (use_beta && !(p.diag & 1)) {
          // beta: the old values of column n + 3 are fetched before column n
          // is combined and stored (two columns' L2 round trips in flight per
          // warp; element by element the loads could not pass the previous
          // stores, and a tile of 16 k-blocks waited ~60 us for its storers)
          double old[BM / 32];
          {
            const int64_t c0 = s_col[swarp];
#pragma unroll
            for (int j = 0; j < BM / 32; ++j)
              old[j] = (c0 >= 0 && roff[j] >= 0) ? Cb[roff[j] + c0] : 0.0;
          }
#pragma unroll 1
          for (int n = swarp; n < BN; n += 3) {
            const int64_t coff = s_col[n];
            const int64_t cnext = n + 3 < BN ? s_col[n + 3] : -1;
            double nxt[BM / 32];
#pragma unroll
            for (int j = 0; j < BM / 32; ++j)
              nxt[j] = (cnext >= 0 && roff[j] >= 0) ? Cb[roff[j] + cnext] : 0.0;
#pragma unroll
            for (int j = 0; j < BM / 32; ++j) {
              const double v = lds64(smem_u32(staging) + stage_off(slane + 32 * j, n));
              if (coff >= 0 && roff[j] >= 0) Cb[roff[j] + coff] = fma(p.beta, old[j], v);
            }
#pragma unroll
            for (int j = 0; j < BM / 32; ++j) old[j] = nxt[j];
          }
        } else {
#pragma unroll 1
          for (int n = swarp; n < BN; n += 3) {
            const int64_t coff = s_col[n];
            double v[BM / 32];
#pragma unroll
            for (int j = 0; j < BM / 32; ++j)
              v[j] = lds64(smem_u32(staging) + stage_off(slane + 32 * j, n));
            if (coff < 0 || (p.diag & 1)) continue;
#pragma unroll
            for (int j = 0; j < BM / 32; ++j)
              if (roff[j] >= 0) Cb[roff[j] + coff] = v[j];
          }
        }
        // the staging loads must have completed before the consumers may
        // overwrite the buffer (see the ring-stage release in the main loop)
        asm volatile("fence.acq_rel.cta;" ::: "memory");
        mbar_arrive(stg_empty);
      }
      return;
    }
    // ============================ producer ============================
    if (USE_TMA && tid != 0) return;
    if (p.gate != nullptr) gate_wait(p);
    LoadIter<SPLITK> li;
    li.template start<USE_TMA>(p);
    uint32_t g = 0;
    const bool pacing = USE_TMA && p.pace != nullptr;
    const uint32_t pace_mask = (1u << p.pace_shift) - 1u;
    bool pace_wait = true;
    uint32_t announced = 0;
#pragma unroll 1
    while (li.valid) {
      if (pacing && g != 0 && (g & pace_mask) == 0) {
        pace_epoch(p, g >> p.pace_shift, pace_wait);
        ++announced;
      }
      const uint32_t s = g % NST;
      mbar_wait(empty0 + 8 * s, ((g / NST) & 1) ^ 1);
      if (USE_TMA && (p.diag & 8) && g >= static_cast<uint32_t>(NST))
        mbar_arrive(full0 + 8 * s);  // TCB_DIAG bit 8 (timing experiment): no reload
      else
        issue_stage<A_KMAJOR, B_KMAJOR, USE_TMA>(p, tmA, tmB, li, s_base + s * STAGE_BYTES,
                                                 full0 + 8 * s, tid);
      if (p.c_pf && li.kb + 1 == li.kb1 && li.kb1 == p.kblocks && li.whole) {
        // beta != 0, C read by a register-path epilogue: prefetch the tile of
        // C into L2 with the tile's last operand loads (one bulk prefetch per
        // column; the consumers are still NST k-blocks behind)
        const double* c0 = p.C + li.m0 + static_cast<int64_t>(li.n0) * p.c_col_str[0];
        const int64_t rows = min(static_cast<int64_t>(BM), p.M - li.m0);
        const uint32_t bytes = static_cast<uint32_t>((rows * 8 + 15) & ~15LL);
        const int cols = static_cast<int>(min(static_cast<int64_t>(BN), p.N - li.n0));
#pragma unroll 1
        for (int j = 0; j < cols; ++j)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c0 + j * p.c_col_str[0]),
                       "r"(bytes)
                       : "memory");
      }
      ++g;
      li.template advance<USE_TMA>(p);
    }
    if (pacing && p.pace_total > announced)  // the epochs this CTA never runs
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p.pace),
                   "l"(static_cast<unsigned long long>(p.pace_total - announced))
                   : "memory");
    if (!USE_TMA) asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }

  // ============================ consumers ============================
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;" ::: "memory");
  const int ctid = tid - PTHREADS;  // 0..255
  const int warp = ctid >> 5, lane = ctid & 31;
  const int wm = warp & 1, wn = warp >> 1;
  const int r = lane >> 2, q = lane & 3;

  // Per-thread swizzle offsets. tile_off splits into a warp-uniform part
  // (compile-time im/in/j terms) and an XOR part that depends on the lane and
  // on two bits of (j, im|in): precompute those 4 lane offsets per operand.
  //   K-major : off[j]                = tile_off<true>(r, kstep_k(j, q))
  //   MN-major: off[(j&1)|(half<<1)]  = tile_off<false>(half*8 + r, kstep_k(j&1, q))
  uint32_t offA[4], offB[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    offA[c] = A_KMAJOR ? tile_off<true>(r, kstep_k(c, q))
                       : tile_off<false>((c >> 1) * 8 + r, kstep_k(c & 1, q));
    offB[c] = B_KMAJOR ? tile_off<true>(r, kstep_k(c, q))
                       : tile_off<false>((c >> 1) * 8 + r, kstep_k(c & 1, q));
  }

  uint32_t gcons = 0;  // k-blocks consumed by this CTA
  uint32_t tcount = 0;  // segments finished by this CTA (staging parity)
  const bool tl = ctid == 0;
  trace_mark(p, 0, tl);
  SegIter<SPLITK> segs;
  segs.init(p);
  int npart = 0;
  int64_t u;
  int kb0, kb1;
#pragma unroll 1
  for (; segs.next(p, u, kb0, kb1); ++tcount) {
    // the staged epilogue needs no unit decode on the consumers
    Unit un{};
    if constexpr (!STAGED) un = decode_unit(p, u);

    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // Staged epilogue woven into the tile's last k-block (see consume_kblock):
    // alpha == 1 only (the scaling would put DMULs between the DMMAs);
    // TCB_DIAG bit 64 keeps the separate store pass for A/B timing.
    const bool weave = STAGED && !p.alpha_ne1 && !(p.diag & 64);
    // likewise a stream-K segment's partial tile into its workspace slot
    const bool weave_sk = SPLITK && (kb0 != 0 || kb1 != p.kblocks) && !(p.diag & 64);
    const int kb_main = (weave || weave_sk) ? kb1 - 1 : kb1;
#pragma unroll 1
    for (int kb = kb0; kb < kb_main; ++kb) {
      const uint32_t stage = gcons % NST;
      mbar_wait(full0 + 8 * stage, (gcons / NST) & 1);
      if (p.trace != nullptr) {  // diagnostics only: one uniform branch per k-block
        if (kb == kb0 && tcount > 0 && tcount <= 8)
          trace_mark(p, 10 + 3 * (static_cast<int>(tcount) - 1), tl);
        if (gcons == 0) trace_mark(p, 1, tl);
        if (gcons == 8) trace_mark(p, 7, tl);
        if (tcount == 2 && kb == kb0 + 4) trace_mark(p, 30, tl);
        if (tcount == 2 && kb == kb0 + 8) trace_mark(p, 31, tl);
      }
      const uint32_t sA = s_base + stage * STAGE_BYTES, sB = sA + STAGE_A;
      consume_kblock<A_KMAJOR, B_KMAJOR, 0>(acc, sA, sB, offA, offB, wm, wn, 0u, nullptr, r, q);
      // Release the stage only once every lane's fragment loads from it have
      // completed: ptxas issues the arrive as soon as the loads are issued
      // (their DMMAs may follow it), and the producer's next TMA write to the
      // stage could then land before a late load reads it (seen as a corrupt
      // warp tile when slow epilogues let the producer run ahead).
      // fence.cta waits for this thread's outstanding loads.
      asm volatile("fence.acq_rel.cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * stage);
      ++gcons;
    }
    if constexpr (STAGED) {
      if (weave) {
        const uint32_t stage = gcons % NST;
        mbar_wait(full0 + 8 * stage, (gcons / NST) & 1);
        if (p.trace != nullptr) {
          if (kb_main == kb0 && tcount > 0 && tcount <= 8)
            trace_mark(p, 10 + 3 * (static_cast<int>(tcount) - 1), tl);
          if (gcons == 0) trace_mark(p, 1, tl);
          if (tcount == 0) trace_mark(p, 2, tl);
          if (tcount < 8) trace_mark(p, 8 + 3 * static_cast<int>(tcount), tl);
        }
        // the storer has drained the previous tile (a tile earlier: no wait in practice)
        mbar_wait(stg_empty, (tcount & 1) ^ 1);
        const uint32_t sA = s_base + stage * STAGE_BYTES, sB = sA + STAGE_A;
        consume_kblock<A_KMAJOR, B_KMAJOR, 1>(acc, sA, sB, offA, offB, wm, wn,
                                              smem_u32(staging), nullptr, r, q);
        asm volatile("fence.acq_rel.cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * stage);
        ++gcons;
        fence_proxy_async_smem();  // the TMA store reads the tile through the async proxy
        mbar_arrive(stg_full);
        if (tcount < 8) trace_mark(p, 9 + 3 * static_cast<int>(tcount), tl);
        continue;
      }
    }
    if constexpr (SPLITK) {
      if (weave_sk) {
        // Stream-K partial (see the separate pass below for the slot layout),
        // stored while the segment's last DMMAs issue; no output tables needed.
        const uint32_t stage = gcons % NST;
        mbar_wait(full0 + 8 * stage, (gcons / NST) & 1);
        if (p.trace != nullptr) {
          if (gcons == 0) trace_mark(p, 1, tl);
          if (tcount == 0) trace_mark(p, 2, tl);
        }
        pdl_wait();  // the previous grid may still read the workspace / counters
        double2* part = reinterpret_cast<double2*>(p.ws) +
                        (2 * static_cast<int64_t>(blockIdx.x) + npart) * (BM * BN / 2) + ctid;
        const uint32_t sA = s_base + stage * STAGE_BYTES, sB = sA + STAGE_A;
        consume_kblock<A_KMAJOR, B_KMAJOR, 2>(acc, sA, sB, offA, offB, wm, wn, 0u, part, r, q);
        asm volatile("fence.acq_rel.cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * stage);
        ++gcons;
        consumer_sync();
        if (npart == 0) trace_mark(p, 3, tl);
        if (ctid == 0)
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.counters + u) : "memory");
        ++npart;
        continue;
      }
    }

    // ------------------------------ epilogue ------------------------------
    if (tcount == 0) trace_mark(p, 2, tl);
    if (tcount < 8) trace_mark(p, 8 + 3 * static_cast<int>(tcount), tl);
    if constexpr (STAGED) {
      // hand the tile to the storers: wait until they drained the previous one,
      // write the raw accumulators ([n][m] with a bank swizzle on m), arrive.
      if (p.alpha_ne1) {
#pragma unroll
        for (int im = 0; im < 8; ++im)
#pragma unroll
          for (int in = 0; in < 4; ++in) {
            acc[im][in][0] *= p.alpha;
            acc[im][in][1] *= p.alpha;
          }
      }
      mbar_wait(stg_empty, (tcount & 1) ^ 1);
      const uint32_t stg = smem_u32(staging);
#pragma unroll
      for (int im = 0; im < 8; ++im)
#pragma unroll
        for (int in = 0; in < 4; ++in)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const uint32_t a = stg + stage_off(wm * 64 + im * 8 + r, wn * 32 + in * 8 + 2 * q + jj);
            asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(acc[im][in][jj]) : "memory");
          }
      fence_proxy_async_smem();  // the TMA store reads these through the async proxy
      mbar_arrive(stg_full);
      if (tcount < 8) trace_mark(p, 9 + 3 * static_cast<int>(tcount), tl);
      continue;
    }
    // Output offsets of this tile's 128 rows and 128 columns, decoded once
    // (one composite index per consumer thread) into shared memory.
    consumer_sync();  // the previous unit's epilogue is done with the tables
    {
      const int i = ctid & 127;
      if (ctid < 128) {
        const int64_t m = static_cast<int64_t>(un.tm) * BM + i;
        s_row[i] = m < p.M ? composite(m, p.c_nrow, p.c_row_ext, p.c_row_str) : -1;
      } else {
        const int64_t n = static_cast<int64_t>(un.tn) * BN + i;
        s_col[i] = n < p.N ? composite(n, p.c_ncol, p.c_col_ext, p.c_col_str) : -1;
      }
    }
    int bc[TCB_MAX_DIMS];
    int64_t oa, ob, oc;
    batch_offsets(p, un.batch, oa, ob, oc, bc);
    double* Cb = p.C + oc;
    const bool use_beta = p.beta != 0.0;

    if (SPLITK && (kb0 != 0 || kb1 != p.kblocks)) {
      // Stream-K: the segment's partial tile goes to workspace slot
      // 2*cta + segment in fragment order (value pair acc[im][in][0..1] of
      // consumer thread t at pair index v*256 + t, v = im*4 + in: one
      // coalesced 16-byte store per pair) and the tile's arrival counter is
      // bumped; the reductions run after all of this CTA's segments, so no
      // CTA waits before it has published everything it owes.
      pdl_wait();  // the previous grid may still read the workspace / counters
      double2* part = reinterpret_cast<double2*>(p.ws) +
                      (2 * static_cast<int64_t>(blockIdx.x) + npart) * (BM * BN / 2);
#pragma unroll
      for (int im = 0; im < 8; ++im)
#pragma unroll
        for (int in = 0; in < 4; ++in)
          __stcg(part + (im * 4 + in) * CTHREADS + ctid,
                 make_double2(acc[im][in][0], acc[im][in][1]));
      // the CTA barrier orders every thread's partial stores before thread 0,
      // whose gpu-scope release (cumulative) then announces them
      consumer_sync();
      if (npart == 0) trace_mark(p, 3, tl);
      if (ctid == 0)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.counters + u) : "memory");
      ++npart;
      continue;
    }

    consumer_sync();
    pdl_wait();
    // Branch-free stores (predicated STG): one unrolled copy per beta mode so
    // the epilogue stays small (it runs once per tile, off the I-cache-hot loop).
    int64_t coff[4][2];
    bool cok[4][2];
#pragma unroll
    for (int in = 0; in < 4; ++in)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        coff[in][jj] = s_col[wn * 32 + in * 8 + 2 * q + jj];
        cok[in][jj] = coff[in][jj] >= 0;
      }
    if (use_beta) {
      store_tile<true>(acc, Cb, s_row, coff, cok, wm, r, p.alpha, p.beta);
    } else {
      store_tile<false>(acc, Cb, s_row, coff, cok, wm, r, p.alpha, p.beta);
    }
  }
  if constexpr (SPLITK) {
    // Reduce this CTA's share of each of its tiles — the pairs in proportion
    // to the k-blocks it computed there — summing the contributors' partials
    // in contributor (= k) order: bit-reproducible, spread over all of them.
    constexpr int PAIRS = BM * BN / 2;
    const bool use_beta = p.beta != 0.0;
    const int my0 = p.sk_start[blockIdx.x], my1 = p.sk_start[blockIdx.x + 1];
    int nred = 0;  // reductions done (trace marks of the first)
#pragma unroll 1
    for (int j = 0; j < 2 && my1 > my0; ++j) {
      // this CTA's tiles: its share's first, then (if it crosses) its last
      const int t = j == 0 ? my0 / p.kblocks : (my1 - 1) / p.kblocks;
      if (j == 1 && t == my0 / p.kblocks) break;
      int p0, p1, first, last;
      if (!sk_reduce_range(p, blockIdx.x, t, PAIRS, p0, p1, first, last)) continue;
      const int S = last - first + 1;
      const Unit un = decode_unit(p, t);
      consumer_sync();  // the previous tile's tables and slots are consumed
      {
        const int i = ctid & 127;
        if (ctid < 128) {
          const int64_t m = static_cast<int64_t>(un.tm) * BM + i;
          s_row[i] = m < p.M ? composite(m, p.c_nrow, p.c_row_ext, p.c_row_str) : -1;
        } else {
          const int64_t n = static_cast<int64_t>(un.tn) * BN + i;
          s_col[i] = n < p.N ? composite(n, p.c_ncol, p.c_col_ext, p.c_col_str) : -1;
        }
        // workspace slot of contributor i: its first partial segment holds
        // tile t unless its share starts inside an earlier tile (a share that
        // starts on a tile boundary opens with a whole tile or with t itself)
        if (ctid < S) {
          const int c = first + ctid;
          const int st0 = p.sk_start[c];
          const bool head_partial = st0 % p.kblocks != 0;
          s_slot[ctid] = 2 * c + ((head_partial && st0 / p.kblocks != t) ? 1 : 0);
        }
      }
      int bc[TCB_MAX_DIMS];
      int64_t oa, ob, oc;
      batch_offsets(p, un.batch, oa, ob, oc, bc);
      double* Cb = p.C + oc;
      if (ctid == 0) {
        const unsigned target = (p.epoch + 1u) * static_cast<unsigned>(S);
        unsigned seen;
        unsigned long long t_start = 0;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(p.counters + t)
                       : "memory");
          if (seen < target) {
            __nanosleep(32);
            const unsigned long long now = wait_clock_ns();
            if (t_start == 0) t_start = now;
            else if (now - t_start > kWaitTrapNs) __trap();  // a contributor never arrived
          }
        } while (seen < target);
      }
      consumer_sync();
      if (nred == 0) trace_mark(p, 4, tl);
      const double2* ws = reinterpret_cast<const double2*>(p.ws);
      // Each thread owns up to RED pairs of the slice and has the partials of
      // up to CB contributors in flight before summing (one L2 round trip for
      // a tile shared by <= CB CTAs instead of one per 4 contributors).
      if (p.diag & 128)  // TCB_DIAG bit 128: the 4-contributor batches (A/B timing)
        sk_reduce_pairs<4>(p, ws, s_slot, s_row, s_col, Cb, S, p0, p1, ctid, use_beta);
      else
        sk_reduce_pairs<SK_RED_CB>(p, ws, s_slot, s_row, s_col, Cb, S, p0, p1, ctid, use_beta);
      if (nred == 0) trace_mark(p, 5, tl);
      ++nred;
    }
  }
  trace_mark(p, 6, tl);
}

// Return the L2 lines of [lo, hi) (128-byte aligned range) to normal
// eviction priority after a launch that loaded them evict_last into the
// persisting set-aside, so no persisting lines outlive the contraction.
__global__ void l2_demote_kernel(uintptr_t lo, int64_t lines) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < lines;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(lo + 128 * i)
                 : "memory");
}

// beta-only update (alpha == 0 or K == 0): C <- beta*C, or 0 when beta == 0
// (reference semantics, src/kernels_reference.cpp:38-45).
__global__ void scale_kernel(Params p) {
  const int64_t total = p.M * p.N * [&] {
    int64_t b = 1;
    for (int i = 0; i < p.nbatch; ++i) b *= p.bat_ext[i];
    return b;
  }();
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t m = e % p.M, n = (e / p.M) % p.N, b = e / (p.M * p.N);
    int bc[TCB_MAX_DIMS];
    int64_t oa, ob, oc;
    batch_offsets(p, b, oa, ob, oc, bc);
    double* dst = p.C + oc + composite(m, p.c_nrow, p.c_row_ext, p.c_row_str) +
                  composite(n, p.c_ncol, p.c_col_ext, p.c_col_str);
    *dst = p.beta == 0.0 ? 0.0 : p.beta * *dst;
  }
}

// ------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// One GEMM index of one operand as a composite of tensor dimensions (first
// fastest): a single (extent, stride) for plain descriptors.
struct Group {
  int n = 0;
  int64_t ext[TCB_MAX_DIMS] = {};
  int64_t str[TCB_MAX_DIMS] = {};
  void one(int64_t e, int64_t st) {
    n = 1;
    ext[0] = e;
    str[0] = st;
  }
  void many(int g, const int64_t* e, const int64_t* st) {
    n = g;
    for (int i = 0; i < g; ++i) {
      ext[i] = e[i];
      str[i] = st[i];
    }
  }
};

// The operand groups of a descriptor.
struct OperandGroups {
  Group am, ak, bk, bn;
};
OperandGroups groups_of(const tcb_gemm_desc& d) {
  OperandGroups g;
  if (d.g_m > 0) g.am.many(d.g_m, d.m_ext, d.a_m_str);
  else g.am.one(d.m, d.a_sm);
  if (d.g_n > 0) g.bn.many(d.g_n, d.n_ext, d.b_n_str);
  else g.bn.one(d.n, d.b_sn);
  if (d.g_k > 0) {
    g.ak.many(d.g_k, d.k_ext, d.a_k_str);
    g.bk.many(d.g_k, d.k_ext, d.b_k_str);
  } else {
    g.ak.one(d.k, d.a_sk);
    g.bk.one(d.k, d.b_sk);
  }
  return g;
}
bool has_groups(const tcb_gemm_desc& d) { return d.g_m > 0 || d.g_n > 0 || d.g_k > 0; }

// Accumulates the dimensions of one 5-D tensor map and its coordinate
// program (see MapProg), then encodes it.
struct MapBuilder {
  struct Dim {
    int64_t ext, str;
    uint32_t box;
    int src;
    int64_t div, mod;
  };
  Dim dims[16];
  int r = 0;
  const char* err = nullptr;

  void push(int64_t ext, int64_t str, uint32_t box, int src, int64_t div, int64_t mod) {
    if (r < 16) dims[r] = Dim{ext, str, box, src, div, mod};
    ++r;
  }
  // Sub-indices [from, n) of group g (index value = source / div0): the first
  // `span` values of each tile are covered by boxes — the whole first
  // sub-index if its extent divides the span (then into the next one), else a
  // span-sized box inside it; the remaining sub-indices get box 1.
  bool push_span(const Group& g, int from, int64_t span, int src, int64_t div0) {
    const int n = g.n - from;
    const int64_t e0 = g.ext[from];
    int used = 1;
    int64_t div = div0;
    if (n == 1 || e0 % span == 0) {
      push(e0, g.str[from], static_cast<uint32_t>(span), src, div, n > 1 ? e0 : 0);
      div *= e0;
    } else if (span % e0 == 0) {
      const int64_t e1 = g.ext[from + 1], b1 = span / e0;
      if (n > 2 && e1 % b1) {
        err = "second extent of a group does not tile the box";
        return false;
      }
      push(e0, g.str[from], static_cast<uint32_t>(e0), src, div, e0);
      push(e1, g.str[from + 1], static_cast<uint32_t>(b1), src, div * e0, n > 2 ? e1 : 0);
      div *= e0 * e1;
      used = 2;
    } else {
      err = "inner extent of a group does not tile the box";
      return false;
    }
    for (int j = from + used; j < g.n; ++j) {
      push(g.ext[j], g.str[j], 1, src, div, j + 1 < g.n ? g.ext[j] : 0);
      div *= g.ext[j];
    }
    return true;
  }
  // sub-indices 1.. of g, box 1
  void push_rest(const Group& g, int src) {
    int64_t div = g.ext[0];
    for (int j = 1; j < g.n; ++j) {
      push(g.ext[j], g.str[j], 1, src, div, j + 1 < g.n ? g.ext[j] : 0);
      div *= g.ext[j];
    }
  }
  // batch dims with a non-zero stride in this tensor, box 1
  void push_batch(const tcb_gemm_desc& d, const int64_t* bstr) {
    int64_t div = 1;
    for (int i = 0; i < d.nbatch; ++i) {
      if (bstr[i] != 0 && d.bat_ext[i] > 1) push(d.bat_ext[i], bstr[i], 1, 2, div, d.bat_ext[i]);
      div *= d.bat_ext[i];
    }
  }
  // Encode (always 5 dims, so the kernel issues a single instruction form,
  // cp.async.bulk.tensor.5d, whatever the rank) and fill the program.
  bool encode(CUtensorMap* map, MapProg* prog, const double* base) {
    auto fn = encode_fn();
    if (!fn) return fail("tensor-map encoder unavailable");
    if (reinterpret_cast<uintptr_t>(base) % 16) return fail("base not 16-byte aligned");
    if (r > 5) return fail("more than 5 tensor-map dimensions");
    cuuint64_t gdim[5], gstr[4];
    cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
    for (int i = 0; i < 5; ++i) {
      const Dim x = i < r ? dims[i] : Dim{1, 2, 1, 3, 1, 0};
      if (x.ext >= (1LL << 31) || x.div >= (1LL << 32) || x.mod >= (1LL << 32))
        return fail("extent above 2^31");
      gdim[i] = static_cast<cuuint64_t>(x.ext);
      box[i] = x.box;
      if (i > 0) {
        const int64_t st = x.ext > 1 ? x.str : 2;  // extent-1 dims: any legal stride
        if (st <= 0 || st % 2 || st * 8 >= (1LL << 40))
          return fail("stride not a positive multiple of 16 bytes");
        gstr[i - 1] = static_cast<cuuint64_t>(st * 8);
      }
      prog->src[i] = x.src;
      prog->div[i] = static_cast<unsigned>(x.div);
      prog->mod[i] = static_cast<unsigned>(x.mod);
    }
    const CUresult res =
        fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(base), gdim, gstr, box,
           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) return fail("tensor-map encoding rejected");
    return true;
  }
  bool fail(const char* w) {
    err = w;
    return false;
  }
};

// Build the tensor map of one operand and its coordinate program.
//   K-major:  [k inner: box 16] [outer: box spanning 128 indices] ...
//   MN-major: [outer % 16: box 16] [k inner: box 16] [outer / 16: box spanning
//             the 8 16-row chunks of the tile] ...
// then the remaining sub-indices (box 1) and the batch dims with a non-zero
// stride (box 1). Span boundaries never cut a box row, so inner extents of
// multi-index groups must be multiples of 16 (and of 128 / divisors of 128
// where they are spanned). One TMA instruction then loads an operand's whole
// stage. MN-major operands with an outer extent that is not a multiple of 16
// (plain descriptors only) use eight 16x16 boxes instead. Returns false with
// `why` set when TMA cannot describe the operand; plain descriptors then fall
// back to cp.async.
bool make_map(CUtensorMap* map, MapProg* prog, const double* base, bool kmajor,
              const Group& outer, const Group& kg, const tcb_gemm_desc& d, const int64_t* bstr,
              const char** why) {
  MapBuilder mb;
  auto fail = [&](const char* w) {
    *why = w;
    return false;
  };
  const Group& lead = kmajor ? kg : outer;
  if (lead.str[0] != 1 && lead.ext[0] > 1) return fail("no unit-stride inner index");
  if (kg.n > 1 && kg.ext[0] % 16) return fail("inner extent of a k group not a multiple of 16");
  prog->nbox = 1;
  if (kmajor) {
    mb.push(kg.ext[0], 1, 16, 1, 1, kg.n > 1 ? kg.ext[0] : 0);
    if (!mb.push_span(outer, 0, BN, 0, 1)) return fail(mb.err);
    mb.push_rest(kg, 1);
    mb.push_batch(d, bstr);
  } else {
    const int64_t e0 = outer.ext[0];
    bool spanned = false;
    // TCB_BOXES8=1 (diagnostics): plain MN-major operands as eight 16x16 boxes
    static const bool boxes8 = getenv("TCB_BOXES8") != nullptr;
    if (e0 % 16 == 0 && !(boxes8 && outer.n == 1)) {
      // the outer group as (outer % 16, outer / 16 = (e0/16, e1, ...))
      Group hi = outer;
      hi.ext[0] = e0 / 16;
      hi.str[0] = 16 * outer.str[0];
      const int from = (hi.ext[0] == 1 && hi.n > 1) ? 1 : 0;
      mb.push(16, 1, 16, 0, 1, 16);
      mb.push(kg.ext[0], kg.str[0], 16, 1, 1, kg.n > 1 ? kg.ext[0] : 0);
      if (!mb.push_span(hi, from, BM / 16, 0, 16)) return fail(mb.err);
      mb.push_rest(kg, 1);
      mb.push_batch(d, bstr);
      spanned = mb.r <= 5;
      if (!spanned && outer.n > 1) return fail("more than 5 tensor-map dimensions");
    } else if (outer.n > 1) {
      return fail("inner extent of a unit-stride group not a multiple of 16");
    }
    if (!spanned) {  // plain operand: eight 16 x 16 boxes per stage
      mb.r = 0;
      prog->nbox = BM / 16;
      mb.push(e0, 1, 16, 0, 1, 0);
      mb.push(kg.ext[0], kg.str[0], 16, 1, 1, kg.n > 1 ? kg.ext[0] : 0);
      mb.push_rest(kg, 1);
      mb.push_batch(d, bstr);
    }
  }
  if (!mb.encode(map, prog, base)) return fail(mb.err);
  prog->kdim = -1;
  if (kg.n == 1)
    for (int i = 0; i < 5; ++i)
      if (prog->src[i] == 1) prog->kdim = i;
  return true;
}

// Tensor map of the output tile for the TMA-store epilogue: [m % 16: box 16]
// [n: box spanning 128] [m / 16: box spanning the 8 chunks] [rest] [batch],
// coordinate sources 0 = m origin, 1 = n origin, 2 = batch index. Its smem
// image (8 boxes of [n 128][m 16], 128B-swizzled) is the staging layout.
// Needs the output rows' inner sub-index unit-stride with an extent that is
// a multiple of 16 (so a box never writes past a row run).
bool make_cmap(CUtensorMap* map, MapProg* prog, double* C, const tcb_gemm_desc& d,
               int rows, const char** why) {
  Group row, col;
  row.many(d.c_nrow, d.c_row_ext, d.c_row_str);
  col.many(d.c_ncol, d.c_col_ext, d.c_col_str);
  if (row.str[0] != 1 || row.ext[0] % 16) {
    *why = "output rows not unit-stride in runs of 16";
    return false;
  }
  MapBuilder mb;
  Group hi = row;
  hi.ext[0] = row.ext[0] / 16;
  hi.str[0] = 16;
  const int from = (hi.ext[0] == 1 && hi.n > 1) ? 1 : 0;
  mb.push(16, 1, 16, 0, 1, 16);
  bool ok = mb.push_span(col, 0, BN, 1, 1) && mb.push_span(hi, from, rows / 16, 0, 16);
  if (ok) {
    mb.push_batch(d, d.bat_sc);
    ok = mb.encode(map, prog, C);
  }
  if (!ok) {
    *why = mb.err;
    return false;
  }
  prog->nbox = 1;
  prog->kdim = -1;
  return true;
}

// Operand layout: MN-major when the outer index's inner sub-index is
// unit-stride (or the outer extent is 1), K-major when k's is.
bool kmajor_of(const Group& outer, const Group& kg) {
  return !(outer.str[0] == 1 || (outer.n == 1 && outer.ext[0] == 1)) && kg.str[0] == 1;
}

template <bool AK, bool BK_, bool TMA>
cudaError_t launch_one(const Params& p, const CUtensorMap& ta, const CUtensorMap& tb,
                       const CUtensorMap& tc, int grid, cudaStream_t s, bool pdl) {
  const bool split = p.splits > 1;
  auto kern = split ? dgemm_dmma_kernel<AK, BK_, TMA, true> : dgemm_dmma_kernel<AK, BK_, TMA, false>;
  const int smem = split ? smem_bytes<false>() : smem_bytes<TMA>();
  // the smem opt-in is a per-device function attribute: remember it per
  // (instantiation, device) — one bit per device, set once
  static std::atomic<uint64_t> attr_set[2];
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_set[split].load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set[split].fetch_or(bit, std::memory_order_release);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  // Split-K CTAs wait on each other, so all of them must be resident: the
  // cooperative attribute guarantees it for a launch on an idle device. Under
  // programmatic dependent launch (which a cooperative launch would
  // serialize) residency follows from grid <= SMs at one CTA per SM: the
  // previous grid's CTAs exit independently of this one, freeing every SM.
  attr[0].id = cudaLaunchAttributeCooperative;
  static const bool no_coop = getenv("TCB_NO_COOP") != nullptr;  // diagnostics
  attr[0].val.cooperative = (p.splits > 1 && !pdl && !no_coop) ? 1 : 0;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p, ta, tb, tc);
  if (e != cudaSuccess && pdl) {  // refused: plain (cooperative) stream order
    cudaGetLastError();
    attr[0].val.cooperative = p.splits > 1 ? 1 : 0;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, p, ta, tb, tc);
  }
  return e;
}

}  // namespace

// Byte ranges [lo, hi) an operand / the output of a descriptor can touch
// (strides are positive; batch offsets included).
std::pair<uintptr_t, uintptr_t> operand_range(const tcb_gemm_desc& d, const double* X, bool left) {
  int64_t last = 0;
  if (has_groups(d)) {
    const int g = left ? d.g_m : d.g_n;
    for (int i = 0; i < g; ++i)
      last += (left ? d.m_ext[i] - 1 : d.n_ext[i] - 1) * (left ? d.a_m_str[i] : d.b_n_str[i]);
    for (int i = 0; i < d.g_k; ++i) last += (d.k_ext[i] - 1) * (left ? d.a_k_str[i] : d.b_k_str[i]);
  } else {
    last += left ? (d.m - 1) * d.a_sm + (d.k - 1) * d.a_sk : (d.k - 1) * d.b_sk + (d.n - 1) * d.b_sn;
  }
  for (int i = 0; i < d.nbatch; ++i) last += (d.bat_ext[i] - 1) * (left ? d.bat_sa[i] : d.bat_sb[i]);
  const uintptr_t lo = reinterpret_cast<uintptr_t>(X);
  return {lo, lo + static_cast<uintptr_t>(last + 1) * 8};
}
std::pair<uintptr_t, uintptr_t> output_range(const tcb_gemm_desc& d, const double* C) {
  int64_t last = 0;
  for (int i = 0; i < d.c_nrow; ++i) last += (d.c_row_ext[i] - 1) * d.c_row_str[i];
  for (int i = 0; i < d.c_ncol; ++i) last += (d.c_col_ext[i] - 1) * d.c_col_str[i];
  for (int i = 0; i < d.nbatch; ++i) last += (d.bat_ext[i] - 1) * d.bat_sc[i];
  const uintptr_t lo = reinterpret_cast<uintptr_t>(C);
  return {lo, lo + static_cast<uintptr_t>(last + 1) * 8};
}

int launch_scale(const tcb_gemm_desc& d, double* C) {
  Params p{};
  p.C = C;
  p.M = d.m;
  p.N = d.n;
  p.c_nrow = d.c_nrow;
  p.c_ncol = d.c_ncol;
  for (int i = 0; i < TCB_MAX_DIMS; ++i) {
    p.c_row_ext[i] = d.c_row_ext[i];
    p.c_row_str[i] = d.c_row_str[i];
    p.c_col_ext[i] = d.c_col_ext[i];
    p.c_col_str[i] = d.c_col_str[i];
    p.bat_ext[i] = d.bat_ext[i];
    p.bat_sa[i] = d.bat_sa[i];
    p.bat_sb[i] = d.bat_sb[i];
    p.bat_sc[i] = d.bat_sc[i];
  }
  p.nbatch = d.nbatch;
  p.beta = d.beta;
  scale_kernel<<<num_sms() * 4, 256, 0, state().stream>>>(p);
  TCB_LAUNCHED();
  return TCB_OK;
}

int check_gemm_groups(const tcb_gemm_desc& d) {
  if (!has_groups(d)) return TCB_OK;
  const OperandGroups g = groups_of(d);
  CUtensorMap t;
  MapProg prog;
  const char* why = nullptr;
  // any 256-byte aligned address: the maps are only encoded, never used
  const double* base = reinterpret_cast<const double*>(uintptr_t{256});
  if (!make_map(&t, &prog, base, kmajor_of(g.am, g.ak), g.am, g.ak, d, d.bat_sa, &why) ||
      !make_map(&t, &prog, base, kmajor_of(g.bn, g.bk), g.bn, g.bk, d, d.bat_sb, &why))
    return set_error(TCB_EUNSUPPORTED, std::string("gemm: index groups: ") + why);
  return TCB_OK;
}

// The thread's k-pacing counter, zeroed (stream-ordered) when first used or
// after a failed launch left its base unknown.
bool make_pace_ready(ThreadState& st) {
  if (!st.pace) {
    if (cudaMalloc(&st.pace, sizeof(unsigned long long)) != cudaSuccess) {
      cudaGetLastError();
      st.pace = nullptr;
      return false;
    }
    st.pace_reset = true;
  }
  if (st.pace_reset) {
    note_stream_op();
    if (cudaMemsetAsync(st.pace, 0, sizeof(unsigned long long), st.stream) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    st.pace_base = 0;
    st.pace_reset = false;
  }
  return true;
}

// Persisting L2 set-aside of at least `bytes` (capped by the device maximum)
// on the current device; false when the device has none or refuses.
bool ensure_persisting_l2(int64_t bytes) {
  static std::mutex mu;
  static int64_t set_bytes[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  std::lock_guard<std::mutex> lock(mu);
  if (set_bytes[dev] >= bytes) return true;
  int maxp = 0;
  if (cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess ||
      maxp <= 0) {
    cudaGetLastError();
    return false;
  }
  const int64_t want = std::min<int64_t>(bytes, maxp);
  if (set_bytes[dev] >= want) return true;
  if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, static_cast<size_t>(want)) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  set_bytes[dev] = want;
  return true;
}

int launch_gemm(const tcb_gemm_desc& d, const double* A, const double* B, double* C) {
  ThreadState& st = state();
  Params p{};
  p.gate = st.gate;  // set by tcb_gemm_gated for this launch only
  p.gate_value = st.gate_value;
  p.A = A;
  p.B = B;
  p.C = C;
  p.M = d.m;
  p.N = d.n;
  p.K = d.k;
  p.a_so = d.a_sm;
  p.a_sk = d.a_sk;
  p.b_so = d.b_sn;
  p.b_sk = d.b_sk;
  p.c_nrow = d.c_nrow;
  p.c_ncol = d.c_ncol;
  int64_t batch = 1;
  for (int i = 0; i < TCB_MAX_DIMS; ++i) {
    p.c_row_ext[i] = d.c_row_ext[i];
    p.c_row_str[i] = d.c_row_str[i];
    p.c_col_ext[i] = d.c_col_ext[i];
    p.c_col_str[i] = d.c_col_str[i];
    p.bat_ext[i] = d.bat_ext[i];
    p.bat_sa[i] = d.bat_sa[i];
    p.bat_sb[i] = d.bat_sb[i];
    p.bat_sc[i] = d.bat_sc[i];
  }
  p.nbatch = d.nbatch;
  for (int i = 0; i < d.nbatch; ++i) batch *= d.bat_ext[i];
  p.alpha = d.alpha;
  p.beta = d.beta;
  p.alpha_ne1 = d.alpha != 1.0;
  p.beta_nz = d.beta != 0.0;
  p.tiles_m = static_cast<int>((d.m + BM - 1) / BM);
  p.tiles_n = static_cast<int>((d.n + BN - 1) / BN);
  const int64_t kblocks = (d.k + BK - 1) / BK;
  if (kblocks >= (1LL << 31)) return set_error(TCB_EUNSUPPORTED, "gemm: K too large");
  p.kblocks = static_cast<int>(kblocks);
  const int64_t tiles = batch * p.tiles_m * p.tiles_n;
  if (d.m >= (1LL << 31) || d.n >= (1LL << 31) || batch >= (1LL << 31) || tiles * 16 >= (1LL << 31))
    return set_error(TCB_EUNSUPPORTED, "gemm: m, n, batch or tile count above 2^31");
  const int sms = num_sms();

  // Stream-K when the tile grid does not fill the SMs evenly:
  //  * tiles < SMs (cfg1-type shapes): G CTAs share all tiles*kblocks
  //    k-blocks in contiguous ranges (>= 4 each);
  //  * more tiles, but the last data-parallel wave would leave > 5 % of the
  //    machine idle (2048x2048: 256 tiles = 1.73 waves of 148): whole tiles
  //    for the full waves (data-parallel phase), then the remaining tiles'
  //    k-blocks shared by all G = SMs CTAs.
  // Shares are shorter than a tile, so a CTA touches at most two tiles of the
  // shared range; a share that crosses a tile boundary is one k-block shorter
  // than its neighbours (its CTA stores two partial tiles).
  const int64_t W_all = tiles * kblocks;
  int G = 1;
  int64_t dp = 0;  // tiles of the data-parallel phase
  if (kblocks >= 8 && W_all < (1LL << 31)) {
    if (tiles < sms) {
      G = static_cast<int>(std::min<int64_t>({static_cast<int64_t>(sms), W_all / 4, SK_MAX}));
      if (G <= tiles) G = 1;
    } else if (sms <= SK_MAX) {
      const int64_t waves = tiles / sms, rem = tiles % sms;
      // TCB_SK_WASTE: idle-fraction threshold of the hybrid (diagnostics). The
      // hybrid's data-parallel phase stores C without the staged epilogue,
      // which costs short-k tiles a few per cent (cfg2 12 %, cfg3 2 %): 5 %
      // by default, 0.4 % for long tiles, whose epilogue is negligible (cfg5:
      // 4096 tiles = 27.7 waves, 1.2 % idle in the last one: 987.9 -> 973.6
      // ms). A hybrid variant with the staged epilogue for its whole tiles (3
      // stages) was measured slower than this one (6 stages) on every long-k
      // shape (cfg5 988 vs 974 ms) and dropped.
      static const double waste_env = getenv("TCB_SK_WASTE") ? atof(getenv("TCB_SK_WASTE")) : -1;
      // Measured (tools/slab_gemm_ab.py, cfg5-shaped 8192^2 GEMMs): the
      // hybrid beats the staged data-parallel launch from 512 k-blocks per
      // tile with beta = 0 (1.0-1.6 %: no last-wave tail, 6-stage ring) and
      // from 768 with beta != 0 (its consumers read C themselves); cfg4 (256
      // k-blocks, 110.7 waves) +0.3 %; cfg3 (64 k-blocks) -2 %.
      static const int64_t long_kb_env = getenv("TCB_SK_LONGKB") ? atoll(getenv("TCB_SK_LONGKB")) : 0;
      const int64_t long_kb = long_kb_env > 0 ? long_kb_env : (d.beta == 0.0 ? 256 : 768);
      const double waste = waste_env >= 0 ? waste_env : (kblocks >= long_kb ? 0.004 : 0.05);
      if (rem != 0 &&
          static_cast<double>(waves + 1) * sms > (1.0 + waste) * static_cast<double>(tiles) &&
          std::min<int64_t>(sms, rem * kblocks / 4) > rem) {
        G = sms;
        dp = waves * sms;
      }
    }
  }
  // CTAs with a share of the shared range (>= 4 k-blocks each); the others
  // only take data-parallel tiles
  const int G_sk = static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>(G, (tiles - dp) * kblocks / 4)));
  const bool streamk = G > 1;
  const int64_t W = (tiles - dp) * kblocks;  // the shared (stream-K) range
  p.splits = streamk ? 2 : 1;  // > 1: the split (stream-K) kernel variant
  p.units = tiles;
  p.work = W;
  p.sk_grid = G;
  p.dp_tiles = static_cast<int>(streamk ? dp : 0);
  int splits = 1;  // reported: most contributors of one tile
  if (streamk) {
    const int64_t base = dp * kblocks;  // table entries are absolute positions
    int64_t pos = 0;
    p.sk_start[0] = static_cast<int>(base);
    for (int c = 0; c < G; ++c) {
      int64_t len = 0;
      if (c < G_sk) {
        len = (W - pos + (G_sk - c) - 1) / (G_sk - c);
        if (c + 1 < G_sk && len > 1 && pos / kblocks != (pos + len - 1) / kblocks) --len;
      }
      pos += len;
      p.sk_start[c + 1] = static_cast<int>(base + pos);
    }
    for (int c = 0; c < G; ++c)  // a share may touch at most two tiles
      if (p.sk_start[c + 1] > p.sk_start[c] &&
          (p.sk_start[c + 1] - 1) / kblocks - p.sk_start[c] / kblocks > 1)
        return set_error(TCB_EUNSUPPORTED, "gemm: stream-K share spans more than two tiles");
    // most contributors of one shared tile (reported), by a two-pointer sweep
    int c = 0;
    for (int64_t t = dp; t < tiles; ++t) {
      while (c + 1 < G && p.sk_start[c + 1] <= t * kblocks) ++c;
      int last = c;
      while (last + 1 < G && p.sk_start[last + 1] <= (t + 1) * kblocks - 1) ++last;
      splits = std::max(splits, last - c + 1);
    }
    const int64_t need = 2LL * G * BM * BN * 8;  // two segment slots per CTA
    if (need > st.ws_bytes) {
      if (st.ws) cudaFree(st.ws);
      st.ws = nullptr;
      st.ws_bytes = 0;
      TCB_CUDA(cudaMalloc(&st.ws, need));
      st.ws_bytes = need;
    }
    // Per-tile arrival counters grow by the tile's contributor count per
    // launch (epoch); they are re-zeroed whenever (tiles, kblocks, G)
    // changes, after a failed launch, on reallocation and long before they
    // could wrap.
    if (tiles > st.counters_n) {
      if (st.counters) cudaFree(st.counters);
      st.counters = nullptr;
      st.counters_n = 0;
      TCB_CUDA(cudaMalloc(&st.counters, tiles * sizeof(unsigned)));
      st.counters_n = tiles;
      st.last_splits = 0;
    }
    if (st.last_splits != G || st.last_tiles != tiles || st.last_kblocks != kblocks ||
        static_cast<int64_t>(st.epoch + 2) * G >= (1LL << 31)) {
      note_stream_op();
      TCB_CUDA(cudaMemsetAsync(st.counters, 0, st.counters_n * sizeof(unsigned), st.stream));
      st.epoch = 0;
    }
    p.ws = static_cast<double*>(st.ws);
    p.counters = st.counters;
    p.epoch = st.epoch;
  }

  const OperandGroups g = groups_of(d);
  const bool a_k = kmajor_of(g.am, g.ak);
  const bool b_k = kmajor_of(g.bn, g.bk);
  CUtensorMap ta, tb;
  std::memset(&ta, 0, sizeof ta);
  std::memset(&tb, 0, sizeof tb);
  const char* why = nullptr;
  const bool tma = make_map(&ta, &p.pa, A, a_k, g.am, g.ak, d, d.bat_sa, &why) &&
                   make_map(&tb, &p.pb, B, b_k, g.bn, g.bk, d, d.bat_sb, &why);
  // index groups are read through the tensor maps only
  if (!tma && has_groups(d)) return set_error(TCB_EUNSUPPORTED, std::string("gemm: index groups: ") + why);
  // staged epilogue: C by TMA store when beta == 0 and the map describes C;
  // beta == 1 (accumulation, the reference loop nest's case) by a TMA
  // reduce-add of the same tile (TCB_NO_CRED=1: the storers' load / DFMA /
  // store path instead, diagnostics)
  CUtensorMap tc;
  std::memset(&tc, 0, sizeof tc);
  static const bool no_cstore = getenv("TCB_NO_CSTORE") != nullptr;  // diagnostics
  static const bool no_cred = getenv("TCB_NO_CRED") != nullptr;
  p.c_tma = 0;
  p.c_red = 0;
  if (tma && !streamk && (d.beta == 0.0 || (d.beta == 1.0 && !no_cred)) && !no_cstore) {
    const char* cwhy = nullptr;
    p.c_tma = make_cmap(&tc, &p.pc, C, d, BM, &cwhy) ? 1 : 0;
    p.c_red = (p.c_tma && d.beta == 1.0) ? 1 : 0;
  }
  // TCB_NO_CPF=1 disables it (diagnostics)
  static const bool no_cpf = getenv("TCB_NO_CPF") != nullptr;
  p.c_pf = (!no_cpf && tma && d.beta != 0.0 && !p.c_tma && d.nbatch == 0 && d.c_nrow == 1 &&
            d.c_ncol == 1 && d.c_row_str[0] == 1 && d.c_col_str[0] % 2 == 0 &&
            reinterpret_cast<uintptr_t>(C) % 16 == 0 && kblocks >= 16)
               ? 1
               : 0;

  const int grid = streamk ? G : static_cast<int>(std::min<int64_t>(tiles, sms));

  // Tile raster. Default: groups of 8 m-tiles per n sweep. When the operands
  // exceed L2 but one side's panels (BM or BN rows x K) fit a 64 MB budget in
  // groups of >= 4, group along the side with fewer tiles and keep that group
  // of panels resident while the other operand streams through (cfg4: groups
  // of 16 of B's 32 panels of 4 MB; A's 512 panels are read twice instead of
  // B being re-read for every group of 8 A panels). TCB_RASTER=m<g>|n<g>
  // overrides (diagnostics).
  p.raster_g = 8;
  p.raster_n = 0;
  {
    const int64_t a_panel = static_cast<int64_t>(BM) * d.k * 8;
    const int64_t b_panel = static_cast<int64_t>(BN) * d.k * 8;
    const int64_t budget = 64LL << 20;
    if ((d.m + d.n) * d.k * 8 > (126LL << 20) && a_panel > budget / 4 &&
        b_panel > budget / 4) {
      // no panel group fits: k-pacing keeps each wave's panels in L2 one
      // k-window at a time, so a wave reads (its m-tiles + its n-tiles)
      // panels; about square waves (12 x 12.3 of 148) minimise that
      p.raster_g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(p.tiles_m, 12)));
    } else if ((d.m + d.n) * d.k * 8 > (126LL << 20)) {
      if (p.tiles_m >= p.tiles_n) {
        const int64_t gn = std::min<int64_t>(p.tiles_n, budget / std::max<int64_t>(1, b_panel));
        if (gn >= 4 && gn < p.tiles_m) {
          p.raster_n = 1;
          p.raster_g = static_cast<int>(gn);
        }
      } else {
        const int64_t gm = std::min<int64_t>(p.tiles_m, budget / std::max<int64_t>(1, a_panel));
        if (gm >= 8) p.raster_g = static_cast<int>(gm);
      }
    }
    static const char* rs = getenv("TCB_RASTER");
    if (rs && (rs[0] == 'm' || rs[0] == 'n') && atoi(rs + 1) > 0) {
      p.raster_n = rs[0] == 'n';
      p.raster_g = atoi(rs + 1);
    }
  }
  // L2 eviction priorities (TMA loads only): a raster that keeps a group of
  // B panels resident while A streams loads B evict_last (cfg4: DRAM reads
  // 9.2 -> 8.7 GB per launch, time unchanged). A stays normal: each A panel
  // slice is read by the group's 16 CTAs within a pacing window, and
  // evict_first on it re-reads A (15 GB). TCB_L2HINT=<a><b>[<c>] with digits
  // 0/1/2 (default / evict_first / evict_last; c = the TMA store of C)
  // overrides (diagnostics).
  p.a_hint = p.b_hint = p.c_hint = 0;
  int64_t resident = 0;  // bytes of the resident panel group
  if (tma && (d.m + d.n) * d.k * 8 > (126LL << 20) && p.raster_n) {
    p.b_hint = 2;
    resident = static_cast<int64_t>(p.raster_g) * BN * d.k * 8;
  }
  {
    static const char* hs = getenv("TCB_L2HINT");
    if (hs && strlen(hs) >= 2) {
      p.a_hint = (hs[0] - '0') % 3;
      p.b_hint = (hs[1] - '0') % 3;
      if (hs[2]) p.c_hint = (hs[2] - '0') % 3;
    }
  }
  // evict_last lines only stay put inside the persisting L2 set-aside
  // (cudaLimitPersistingL2CacheSize, 0 by default). TCB_L2PERSIST=1 (or =<MB>)
  // grows it to the resident group (capped by the device) and a demotion
  // kernel after the launch returns the group's lines to normal priority, so
  // no persisting lines outlive the contraction. Off by default: measured on
  // cfg4 it cuts DRAM reads from 8.7 to 4.8 GB per launch but costs 0.6 % of
  // the launch time (any set-aside size, 16-64 MB), and time is the metric.
  bool demote = false;
  if (p.b_hint == 2 && resident > 0) {
    static const char* pe = getenv("TCB_L2PERSIST");
    static const int64_t mb = pe ? atoll(pe) : 0;
    static const bool no_demote = getenv("TCB_NO_L2DEMOTE") != nullptr;  // diagnostics
    if (mb > 0) {
      const int64_t want = mb > 1 ? std::min<int64_t>(resident, mb << 20) : resident;
      demote = ensure_persisting_l2(want) && !no_demote;
    }
  }

  // k-pacing (see Params) for long-k launches through TMA: every CTA issues
  // at least 8 epochs of 32 k-blocks and tiles have >= 128 k-blocks.
  // TCB_NO_PACE=1 disables it (diagnostics).
  p.pace = nullptr;
  p.kflip = 0;
  {
    static const bool no_pace = getenv("TCB_NO_PACE") != nullptr;
    int64_t maxkb = 0;  // most k-blocks any CTA issues
    if (streamk) {
      for (int c = 0; c < G; ++c) {
        const int64_t dpt = c < dp ? (dp - 1 - c) / G + 1 : 0;
        maxkb = std::max<int64_t>(maxkb, dpt * kblocks + p.sk_start[c + 1] - p.sk_start[c]);
      }
    } else {
      maxkb = (tiles + grid - 1) / grid * kblocks;
    }
    // TCB_PACE=<shift>,<slack> (diagnostics): epoch 2^shift k-blocks, slack in epochs
    static const char* pe = getenv("TCB_PACE");
    static const int kShift = pe ? std::max(1, atoi(pe)) : 4;
    static const int kSlack = (pe && strchr(pe, ',')) ? std::max(1, atoi(strchr(pe, ',') + 1)) : 1;
    if (!no_pace && tma && kblocks >= 128 && maxkb >= (8LL << kShift) &&
        make_pace_ready(st)) {
      static const bool no_flip = getenv("TCB_NO_KFLIP") != nullptr;
      p.kflip = no_flip ? 0 : 1;
      p.pace = st.pace;
      p.pace_base = st.pace_base;
      p.pace_shift = kShift;
      p.pace_slack = kSlack;
      p.pace_grid = grid;
      p.pace_total = static_cast<unsigned>((maxkb + (1 << kShift) - 1) >> kShift);
    }
  }
  // Programmatic dependent launch when the operations on our own stream since
  // the last serialized launch are all GEMMs and none of their outputs
  // overlaps this one's operands (read before griddepcontrol.wait).
  // TCB_NO_PDL=1 disables it.
  static const bool no_pdl = getenv("TCB_NO_PDL") != nullptr;
  const auto [alo, ahi] = operand_range(d, A, true);
  const auto [blo, bhi] = operand_range(d, B, false);
  const bool pdl = !no_pdl && st.pdl_ok && st.stream == st.own_stream &&
                   st.pdl_clear(alo, ahi) && st.pdl_clear(blo, bhi);
  // TCB_TRACE=<file>: append per-CTA phase timestamps of this launch (diagnostics)
  static const char* trace_path = getenv("TCB_TRACE");
  unsigned long long* trace = nullptr;
  if (trace_path) {
    TCB_CUDA(cudaMalloc(&trace, grid * 32 * sizeof(unsigned long long)));
    TCB_CUDA(cudaMemsetAsync(trace, 0, grid * 32 * sizeof(unsigned long long), st.stream));
  }
  p.trace = trace;
  if (trace) note_stream_op();
  static const int diag = getenv("TCB_DIAG") ? atoi(getenv("TCB_DIAG")) : 0;
  p.diag = diag;
  cudaError_t e;
  if (tma) {
    if (a_k && b_k) e = launch_one<true, true, true>(p, ta, tb, tc, grid, st.stream, pdl);
    else if (a_k) e = launch_one<true, false, true>(p, ta, tb, tc, grid, st.stream, pdl);
    else if (b_k) e = launch_one<false, true, true>(p, ta, tb, tc, grid, st.stream, pdl);
    else e = launch_one<false, false, true>(p, ta, tb, tc, grid, st.stream, pdl);
  } else {
    if (a_k && b_k) e = launch_one<true, true, false>(p, ta, tb, tc, grid, st.stream, pdl);
    else if (a_k) e = launch_one<true, false, false>(p, ta, tb, tc, grid, st.stream, pdl);
    else if (b_k) e = launch_one<false, true, false>(p, ta, tb, tc, grid, st.stream, pdl);
    else e = launch_one<false, false, false>(p, ta, tb, tc, grid, st.stream, pdl);
  }
  if (e != cudaSuccess) {
    st.last_splits = 0;
    if (p.pace) st.pace_reset = true;
    return cuda_fail(e, "dgemm_dmma launch");
  }
  ++st.launches;
  if (p.pace) st.pace_base += static_cast<unsigned long long>(p.pace_total) * grid;
  {
    // outputs of the PDL chain: a fully serialized launch starts a new chain
    // (everything before it has completed); a PDL launch extends it
    const auto [clo, chi] = output_range(d, C);
    st.pdl_add(clo, chi, pdl);
    st.pdl_ok = true;
  }
  if (demote) {
    const auto [blo, bhi] = operand_range(d, B, false);
    const uintptr_t lo = blo & ~static_cast<uintptr_t>(127);
    const int64_t lines = static_cast<int64_t>((bhi - lo + 127) / 128);
    l2_demote_kernel<<<4 * sms, 256, 0, st.stream>>>(lo, lines);
    note_stream_op();  // the next GEMM starts a new PDL chain after it
    ++st.launches;
  }
  if (trace) {
    note_stream_op();
    std::vector<unsigned long long> h(static_cast<size_t>(grid) * 32);
    TCB_CUDA(cudaMemcpyAsync(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost, st.stream));
    TCB_CUDA(cudaStreamSynchronize(st.stream));
    cudaFree(trace);
    if (FILE* f = fopen(trace_path, "a")) {
      fprintf(f, "{\"m\":%lld,\"n\":%lld,\"k\":%lld,\"splits\":%d,\"grid\":%d,\"t\":[",
              static_cast<long long>(d.m), static_cast<long long>(d.n),
              static_cast<long long>(d.k), splits, grid);
      for (size_t i = 0; i < h.size(); ++i) fprintf(f, "%s%llu", i ? "," : "", h[i]);
      fprintf(f, "]}\n");
      fclose(f);
    }
  }
  if (streamk) {
    ++st.epoch;  // each tile's counter now holds epoch * (its contributor count)
    st.last_splits = G;
    st.last_tiles = tiles;
    st.last_kblocks = kblocks;
  }
  st.last_info.path = tma ? 0 : 1;
  st.last_info.splits = splits;
  st.last_info.units = streamk ? dp + W : tiles;
  st.last_info.grid = grid;
  st.last_info.launches = demote ? 2 : 1;
  return TCB_OK;
}

}  // namespace tcb
