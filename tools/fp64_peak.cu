// fp64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) and DFMA
// throughput with register-resident operands. Prints one JSON line per case.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

// NACC accumulators, each updated CHAIN times in a row (k-chained issue order)
template <int NACC, int CHAIN>
__global__ void dmma_chain(double* out, int iters) {
  double a[CHAIN], b[CHAIN];
#pragma unroll
  for (int i = 0; i < CHAIN; ++i) { a[i] = 1.0 + (threadIdx.x + i) * 1e-9; b[i] = 1.0 - i * 1e-9; }
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
#pragma unroll
      for (int k = 0; k < CHAIN; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a[k]), "d"(b[k]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]),
                     "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <typename K>
int run(const char* name, K kern, int threads, int blocks_per_sm, int iters,
        double flop_per_thread_iter, double* out, int nsm) {
  int grid = nsm * blocks_per_sm;
  kern<<<grid, threads>>>(out, iters / 10);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, threads>>>(out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double flops = flop_per_thread_iter * (double)threads * grid * iters;
  printf("{\"case\": \"%s\", \"threads\": %d, \"blocks_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n",
         name, threads, blocks_per_sm, best, flops / best / 1e9);
  return 0;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", nsm, clk);
  double* out;
  CK(cudaMalloc(&out, 1 << 20));
  const int it = 20000;
  // m8n8k4: 8*8*4 FMA per warp = 256 FMA = 512 flop per warp -> 16 flop per thread
  for (int bps : {1, 2, 4, 8})
    run("dmma_m8n8k4_acc8", dmma_m8n8k4<8>, 128, bps, it, 8 * 16.0, out, nsm);
  for (int bps : {1, 2, 4})
    run("dmma_m8n8k4_acc16", dmma_m8n8k4<16>, 128, bps, it, 16 * 16.0, out, nsm);
  run("dmma_m8n8k4_acc4_256t", dmma_m8n8k4<4>, 256, 2, it, 4 * 16.0, out, nsm);
  run("dmma_m8n8k4_acc1_1024t", dmma_m8n8k4<1>, 1024, 1, it, 1 * 16.0, out, nsm);
  for (int bps : {1, 2}) {
    run("dmma_m8n8k4_acc8_chain2", dmma_chain<8, 2>, 128, bps, it / 2, 16 * 16.0, out, nsm);
    run("dmma_m8n8k4_acc8_chain4", dmma_chain<8, 4>, 128, bps, it / 4, 32 * 16.0, out, nsm);
    run("dmma_m8n8k4_acc16_chain4", dmma_chain<16, 4>, 128, bps, it / 4, 64 * 16.0, out, nsm);
    run("dmma_m8n8k4_acc32_chain1", dmma_chain<32, 1>, 128, bps, it / 4, 32 * 16.0, out, nsm);
  }
  // m16n8k16: 16*8*16 = 2048 FMA per warp -> 128 flop per thread
  for (int bps : {1, 2, 4})
    run("dmma_m16n8k16_acc4", dmma_m16n8k16<4>, 128, bps, it / 4, 4 * 128.0, out, nsm);
  for (int bps : {1, 2, 4, 8})
    run("dfma_acc8", dfma_loop<8>, 256, bps, it, 8 * 2.0, out, nsm);
  return 0;
}
