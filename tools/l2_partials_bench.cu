// Microbenchmark (development aid): the stream-K fix-up's memory pattern.
// G CTAs each write one 128 KB partial tile to L2 and then read back a 1/S
// slice of S partials, as dgemm_dmma's split-K epilogue does; variants:
//   mode 0: STG.128 from registers (__stcg), LDG.128 (__ldcg) reduction
//   mode 1: registers -> smem, one cp.async.bulk smem -> global store of 128 KB
// Prints per-phase times (us, median/max over CTAs) for bytes per CTA of
// 32/64/128 KB. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// tools/l2_partials_bench tools/l2_partials_bench.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) kern(double2* ws, int pairs, int S, unsigned long long* tr,
                                               unsigned* bar, unsigned epoch) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int t = threadIdx.x;
  double2 v[64];
  const int per = pairs / 256;  // pairs per thread
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = make_double2(i + t, blockIdx.x);
  __syncthreads();
  unsigned long long t0 = gtime();
  double2* part = ws + static_cast<long long>(blockIdx.x) * pairs;
  if (MODE == 0) {
#pragma unroll
    for (int i = 0; i < 64; ++i)
      if (i < per) __stcg(part + i * 256 + t, v[i]);
  } else {
    double2* s = reinterpret_cast<double2*>(sm);
#pragma unroll
    for (int i = 0; i < 64; ++i)
      if (i < per) s[i * 256 + t] = v[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(sm));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(part),
                   "r"(sa), "r"(pairs * 16) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }
  __syncthreads();
  unsigned long long t1 = gtime();
  // grid barrier
  if (t == 0) {
    __threadfence();
    atomicAdd(bar, 1);
    const unsigned target = (epoch + 1) * gridDim.x;
    while (atomicAdd(bar, 0) < target) {}
  }
  __syncthreads();
  unsigned long long t2 = gtime();
  // reduction: this CTA sums slice [b*pairs/S ...) of S partials of CTAs (b/S)*S ..
  const int g0 = (blockIdx.x / S) * S;
  const int lo = (blockIdx.x % S) * (pairs / S), hi = lo + pairs / S;
  double acc = 0;
  for (int p = lo + t; p < hi; p += 256) {
    double2 s = make_double2(0, 0);
    for (int c = 0; c < S; ++c) {
      double2 x = __ldcg(ws + static_cast<long long>(g0 + c) * pairs + p);
      s.x += x.x; s.y += x.y;
    }
    acc += s.x + s.y;
  }
  if (acc == 123.456) ws[0] = make_double2(acc, acc);
  __syncthreads();
  unsigned long long t3 = gtime();
  if (t == 0) {
    tr[blockIdx.x * 4 + 0] = t0; tr[blockIdx.x * 4 + 1] = t1;
    tr[blockIdx.x * 4 + 2] = t2; tr[blockIdx.x * 4 + 3] = t3;
  }
}

int main() {
  const int G = 148, S = 9;
  double2* ws; unsigned long long* tr; unsigned* bar;
  cudaMalloc(&ws, 148ull * 8192 * 16);
  cudaMalloc(&tr, G * 4 * 8);
  cudaMalloc(&bar, 4);
  cudaMemset(bar, 0, 4);
  cudaFuncSetAttribute(kern<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  unsigned epoch = 0;
  for (int mode = 0; mode < 2; ++mode)
    for (int kb : {32, 64, 128}) {
      const int pairs = kb * 1024 / 16;
      for (int rep = 0; rep < 5; ++rep) {
        if (mode == 0) kern<0><<<G, 256, 0>>>(ws, pairs, S, tr, bar, epoch++);
        else kern<1><<<G, 256, 140 * 1024>>>(ws, pairs, S, tr, bar, epoch++);
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      std::vector<unsigned long long> h(G * 4);
      cudaMemcpy(h.data(), tr, G * 4 * 8, cudaMemcpyDeviceToHost);
      std::vector<double> st, wt, rd;
      for (int b = 0; b < G; ++b) {
        st.push_back((h[b * 4 + 1] - h[b * 4 + 0]) / 1965.0);
        wt.push_back((h[b * 4 + 2] - h[b * 4 + 1]) / 1965.0);
        rd.push_back((h[b * 4 + 3] - h[b * 4 + 2]) / 1965.0);
      }
      auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
      auto mx = [](std::vector<double> v) { return *std::max_element(v.begin(), v.end()); };
      printf("mode %d  %3d KB/CTA: store med %.2f max %.2f | barrier med %.2f | reduce(S=%d) med %.2f max %.2f us\n",
             mode, kb, med(st), mx(st), med(wt), S, med(rd), mx(rd));
    }
  return 0;
}
