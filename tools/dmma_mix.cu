// DMMA issue-mix microbenchmark (sm_100a): the GEMM consumer's inner loop
// stripped to its instruction mix — per k-step 12 fragment loads (LDS.64,
// conflict-free) feeding 32 DMMA.8x8x4 on 32 independent accumulators — with
// 8 warps per CTA (2 per SM sub-partition), one CTA per SM, no global traffic.
// The fraction of peak it reaches bounds what the real main loop can reach.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_mix dmma_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int LOADS, int BARRIER = 0>
__global__ void __launch_bounds__(256, 1) mix(double* out, int iters) {
  __shared__ double sm[4096];
  __shared__ unsigned long long bar[2];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(&bar[0]))), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(&bar[1]))), "r"((1 << 20) - 1));
  }
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(sm)) + lane * 8;
  const unsigned b0 = static_cast<unsigned>(__cvta_generic_to_shared(&bar[0]));
  const unsigned b1 = static_cast<unsigned>(__cvta_generic_to_shared(&bar[1]));
  for (int it = 0; it < iters; ++it) {
    if (BARRIER && (it & 3) == 0) {
      // the consumer's per-k-block handshake: wait on a completed phase,
      // then (lane 0) arrive on a barrier that never completes
      asm volatile(
          "{\n .reg .pred p;\n"
          "W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n"
          ::"r"(b0), "r"(1) : "memory");
      __syncwarp();
      if ((threadIdx.x & 31) == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b1) : "memory");
    }
    double a[8], b[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (LOADS) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a[i]) : "r"(base + ((it * 12 + i) & 15) * 256));
      else a[i] = 1.0 + i;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (LOADS) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(b[i]) : "r"(base + ((it * 12 + 8 + i) & 15) * 256));
      else b[i] = 2.0 + i;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]) : "d"(a[i]), "d"(b[j]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int LOADS, int BARRIER = 0>
void run(const char* name, int nsm, double* out) {
  const int iters = 20000;
  mix<LOADS, BARRIER><<<nsm, 256>>>(out, 100);
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
    mix<LOADS, BARRIER><<<nsm, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 512.0 * 32 * 8 * (double)nsm * iters;  // per warp-DMMA 512 flop
  printf("{\"case\": \"%s\", \"tflops\": %.3f}\n", name, flops / best / 1e9);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  run<0>("32 DMMA per k-step, no loads", nsm, out);
  run<1>("32 DMMA + 12 LDS.64 per k-step", nsm, out);
  run<1, 1>("... + mbarrier wait/arrive every 4 k-steps", nsm, out);
  return 0;
}
