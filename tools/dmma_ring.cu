// DMMA main-loop microbenchmark (sm_100a, development aid): the GEMM's
// consumer loop with its real synchronisation — a ring of NST shared-memory
// stages with full/empty mbarriers, one producer thread refilling each stage
// with a 32 KB bulk copy from an L2-resident buffer (the TMA's smem write
// traffic), consumers waiting on `full`, running 4 k-steps of fragment loads
// + DMMA, fencing and releasing the stage — for two consumer layouts:
//   8 warps x (64 x 32) warp tiles: 12 LDS.64 + 32 DMMA per k-step (the kernel)
//  16 warps x (32 x 32) warp tiles:  8 LDS.64 + 16 DMMA per k-step
// Prints TFLOP/s per case (no global writes; one CTA per SM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_ring tools/dmma_ring.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int STAGE = 32768;

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

template <int NW, int IM, int IN, int NST, bool FENCE, bool COPY, int CB = STAGE>
__global__ void __launch_bounds__(NW * 32 + 32, 1) ring(const double* src, double* out, int kblocks) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  const unsigned full0 = base + NST * STAGE, empty0 = full0 + 8 * NST;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(full0 + 8 * s), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(empty0 + 8 * s), "r"(NW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < NST * STAGE / 8; i += blockDim.x)
    reinterpret_cast<double*>(sm)[i] = 1.0 + (i & 255) * 1e-9;
  __syncthreads();
  if (tid >= NW * 32) {  // producer warp
    if (tid != NW * 32) return;
    for (int g = 0; g < kblocks; ++g) {
      const int s = g % NST;
      mbar_wait(empty0 + 8 * s, ((g / NST) & 1) ^ 1);
      if (COPY) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full0 + 8 * s),
                     "r"(CB) : "memory");
        const double* g0 = src + static_cast<size_t>((blockIdx.x * 7 + g) & 63) * (STAGE / 8);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                base + s * STAGE),
            "l"(g0), "r"(CB), "r"(full0 + 8 * s)
            : "memory");
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full0 + 8 * s) : "memory");
      }
    }
    return;
  }
  const int lane = tid & 31, warp = tid >> 5;
  double acc[IM][IN][2];
#pragma unroll
  for (int i = 0; i < IM; ++i)
#pragma unroll
    for (int j = 0; j < IN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // conflict-free 8-byte lane addresses inside a stage (A half / B half)
  const unsigned la = (warp * 64 + lane) * 8 % 16384, lb = 16384 + (warp * 32 + lane) * 8 % 16384;
  for (int g = 0; g < kblocks; ++g) {
    const int s = g % NST;
    mbar_wait(full0 + 8 * s, (g / NST) & 1);
    const unsigned sa = base + s * STAGE;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double a[IM], b[IN];
#pragma unroll
      for (int i = 0; i < IM; ++i)
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a[i]) : "r"(sa + la + ((j * IM + i) & 31) * 512));
#pragma unroll
      for (int i = 0; i < IN; ++i)
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(b[i]) : "r"(sa + lb + ((j * IN + i) & 15) * 512 % 16384));
#pragma unroll
      for (int i = 0; i < IM; ++i)
#pragma unroll
        for (int jj = 0; jj < IN; ++jj)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[i][jj][0]), "+d"(acc[i][jj][1]) : "d"(a[i]), "d"(b[jj]));
    }
    if (FENCE) asm volatile("fence.acq_rel.cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * s) : "memory");
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < IM; ++i)
#pragma unroll
    for (int j = 0; j < IN; ++j) t += acc[i][j][0] + acc[i][j][1];
  if (t == 1234.5) out[tid] = t;
}

template <int NW, int IM, int IN, int NST, bool FENCE, bool COPY, int CB = STAGE>
void run(const char* name, int nsm, const double* src, double* out) {
  auto k = ring<NW, IM, IN, NST, FENCE, COPY, CB>;
  const int smem = NST * STAGE + 16 * NST + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int kb = 4000;
  k<<<nsm, NW * 32 + 32, smem>>>(src, out, 50);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("{\"case\": \"%s\", \"error\": \"%s\"}\n", name, cudaGetErrorString(cudaGetLastError()));
    return;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k<<<nsm, NW * 32 + 32, smem>>>(src, out, kb);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  // a k-block = (NW warps x IM*8 x IN*8) x 16 per CTA
  const double flops = 2.0 * NW * IM * 8 * IN * 8 * 16 * (double)nsm * kb;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k);
  printf("{\"case\": \"%s\", \"tflops\": %.3f, \"regs\": %d, \"spill\": %zu}\n", name,
         flops / best / 1e9, fa.numRegs, fa.localSizeBytes);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *src, *out;
  cudaMalloc(&src, 64 * STAGE);
  cudaMemset(src, 0, 64 * STAGE);
  cudaMalloc(&out, 1 << 20);
  run<8, 8, 4, 3, true, true>("8w 64x32 (CTA 128x128), 3 st, fence, copy 32K", nsm, src, out);
  run<8, 8, 4, 6, true, true>("8w 64x32 (CTA 128x128), 6 st, fence, copy 32K", nsm, src, out);
  run<16, 4, 4, 3, true, true>("16w 32x32 (CTA 128x128), 3 st, fence, copy 32K", nsm, src, out);
  run<8, 8, 2, 6, true, true, 24576>("8w 64x16 (CTA 128x64), 6 st, fence, copy 24K", nsm, src, out);
  run<8, 4, 4, 6, true, true, 24576>("8w 32x32 (CTA 128x64), 6 st, fence, copy 24K", nsm, src, out);
  run<8, 4, 2, 6, true, true, 16384>("8w 32x16 (CTA 64x64), 6 st, fence, copy 16K", nsm, src, out);
  run<4, 8, 4, 6, true, true, 24576>("4w 64x32 (CTA 128x64), 6 st, fence, copy 24K", nsm, src, out);
  return 0;
}
