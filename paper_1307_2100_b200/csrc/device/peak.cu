// fp64 roofline denominator, measured live: DMMA (mma.sync m8n8k4 f64)
// throughput with register-resident operands, 2 CTAs x 4 warps per SM, 8
// independent accumulators per warp (enough to saturate the pipe; see
// tools/fp64_peak.cu for the sweep). MEASURED_PEAKS.json has no fp64 entry,
// so bench.py reports its fraction against this number.
#include "tcb_internal.cuh"

namespace tcb {
namespace {

__global__ void __launch_bounds__(128) dmma_peak_kernel(double* sink, int iters) {
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234567.0) sink[threadIdx.x] = s;  // keep the work alive
}

}  // namespace
}  // namespace tcb

using namespace tcb;

extern "C" int tcb_fp64_peak(double* tflops) {
  int rc = ensure_init();
  if (rc != TCB_OK) return rc;
  ThreadState& st = state();
  double* sink = nullptr;
  TCB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sink), 128 * 8, st.stream));
  const int grid = num_sms() * 2, iters = 20000;
  dmma_peak_kernel<<<grid, 128, 0, st.stream>>>(sink, iters / 10);  // warm-up
  TCB_LAUNCHED();
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    TCB_CUDA(cudaEventRecord(st.ev0, st.stream));
    dmma_peak_kernel<<<grid, 128, 0, st.stream>>>(sink, iters);
    TCB_LAUNCHED();
    TCB_CUDA(cudaEventRecord(st.ev1, st.stream));
    TCB_CUDA(cudaEventSynchronize(st.ev1));
    float ms = 0.f;
    TCB_CUDA(cudaEventElapsedTime(&ms, st.ev0, st.ev1));
    best = ms < best ? ms : best;
  }
  cudaFreeAsync(sink, st.stream);
  // 8 DMMA per warp-iteration, 512 flop per DMMA.8x8x4
  const double flops = 512.0 * 8.0 * (128 / 32) * static_cast<double>(grid) * iters;
  if (tflops) *tflops = flops / (best * 1e-3) / 1e12;
  return TCB_OK;
}
