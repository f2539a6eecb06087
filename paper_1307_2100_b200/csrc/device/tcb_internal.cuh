// Internal helpers shared by the device translation units of libtcb200.so.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "tcb.h"

namespace tcb {

// Per (host thread, device) state: the device's stream for this thread, a
// grow-only workspace (split-K partials + per-tile counters), PDL bookkeeping.
// A thread that alternates between devices (tcb_init(d) before each call)
// keeps one of these per device, so nothing is dropped or leaked on a switch.
struct ThreadState {
  int device = -1;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;  // own_stream or a caller stream
  void* ws = nullptr;             // split-K partials
  int64_t ws_bytes = 0;
  unsigned* counters = nullptr;   // split-K per-tile arrival counters
  int64_t counters_n = 0;
  unsigned epoch = 0;             // split-K launches since the counters were zeroed
  int last_splits = 0;             // (G, tiles, kblocks) of the last stream-K launch
  int64_t last_tiles = 0;
  int64_t last_kblocks = 0;
  const unsigned long long* gate = nullptr;  // tcb_gemm_gated: the next launch's gate
  unsigned long long gate_value = 0;
  unsigned long long* pace = nullptr;  // k-pacing counter (monotonic across launches)
  unsigned long long pace_base = 0;    // its value once every earlier launch has finished
  bool pace_reset = true;              // re-zero before the next paced launch
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // tcb_timer_start / tcb_timer_stop
  cudaEvent_t order = nullptr;                // tcb_set_stream's hand-over
  int64_t launches = 0;
  // Programmatic dependent launch: true while the operations enqueued on the
  // thread's own stream since the last fully serialized launch are all DMMA
  // GEMMs (a PDL chain). The intervals [pdl_lo[i], pdl_hi[i]) cover the
  // union of their outputs: a GEMM launched with PDL may issue its operand
  // loads while ANY earlier GEMM of the chain still runs (each one lets its
  // dependent start once its own CTAs are resident), so its operands must
  // avoid every output of the chain, not just the last one. Up to 8 disjoint
  // intervals are kept (repeated calls rotating over several output buffers
  // stay chained); beyond that they collapse into one bounding interval.
  // Every other stream operation clears the chain.
  static constexpr int kPdlRanges = 8;
  bool pdl_ok = false;
  int pdl_n = 0;
  uintptr_t pdl_lo[kPdlRanges] = {}, pdl_hi[kPdlRanges] = {};
  bool pdl_clear(uintptr_t lo, uintptr_t hi) const {  // [lo, hi) misses every chain output
    for (int i = 0; i < pdl_n; ++i)
      if (lo < pdl_hi[i] && pdl_lo[i] < hi) return false;
    return true;
  }
  void pdl_add(uintptr_t lo, uintptr_t hi, bool extend) {
    if (!extend) pdl_n = 0;
    for (int i = 0; i < pdl_n; ++i)
      if (lo <= pdl_hi[i] && pdl_lo[i] <= hi) {  // overlapping or adjacent: merge
        pdl_lo[i] = lo < pdl_lo[i] ? lo : pdl_lo[i];
        pdl_hi[i] = hi > pdl_hi[i] ? hi : pdl_hi[i];
        return;
      }
    if (pdl_n == kPdlRanges) {  // collapse into one bounding interval
      for (int i = 1; i < pdl_n; ++i) {
        pdl_lo[0] = pdl_lo[i] < pdl_lo[0] ? pdl_lo[i] : pdl_lo[0];
        pdl_hi[0] = pdl_hi[i] > pdl_hi[0] ? pdl_hi[i] : pdl_hi[0];
      }
      pdl_n = 1;
      pdl_lo[0] = lo < pdl_lo[0] ? lo : pdl_lo[0];
      pdl_hi[0] = hi > pdl_hi[0] ? hi : pdl_hi[0];
      return;
    }
    pdl_lo[pdl_n] = lo;
    pdl_hi[pdl_n] = hi;
    ++pdl_n;
  }
  tcb_gemm_info last_info{};
};

constexpr int kMaxDevices = 16;
ThreadState& state();            // the calling thread's state for its current device
std::string& thread_error();     // the calling thread's last error text
int set_error(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
int ensure_init();  // lazily binds device 0 when tcb_init was not called

#define TCB_CUDA(call)                                        \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return ::tcb::cuda_fail(e_, #call); \
  } while (0)

#define TCB_LAUNCHED()                                                       \
  do {                                                                       \
    cudaError_t e_ = cudaGetLastError();                                     \
    if (e_ != cudaSuccess) return ::tcb::cuda_fail(e_, "kernel launch");     \
    ++::tcb::state().launches;                                               \
    ::tcb::state().pdl_ok = false;                                           \
  } while (0)

// A non-GEMM operation was enqueued on `stream` (the current one when null).
inline void note_stream_op(cudaStream_t stream = nullptr) {
  ThreadState& st = state();
  if (stream == nullptr || stream == st.stream) st.pdl_ok = false;
}

// Device-side waits on another grid, process or stream give up after this
// long and trap (the kernel fails with an error instead of hanging the GPU):
// a peer rank that died, an upload that never came.
#ifdef __CUDACC__
constexpr unsigned long long kWaitTrapNs = 60ull * 1000 * 1000 * 1000;
__device__ __forceinline__ unsigned long long wait_clock_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

// Device-side launchers (implemented in the .cu files).
int launch_gemm(const tcb_gemm_desc& d, const double* A, const double* B, double* C);
// Index-group descriptors: can the operand tensor maps describe them?
int check_gemm_groups(const tcb_gemm_desc& d);
int launch_permute(int rank, const int64_t* ext, const int64_t* src_str, const double* src,
                   double* dst);
int launch_gemv(const tcb_gemm_desc& d, const double* A, const double* B, double* C);
int launch_scale(const tcb_gemm_desc& d, double* C);
int num_sms();
// cuStreamWriteValue64 / cuStreamWaitValue64 (driver entry points; null when
// the driver lacks them or the device cannot do 64-bit stream memory ops)
int stream_write_value(cudaStream_t s, uint64_t* addr, uint64_t value);
int stream_wait_value(cudaStream_t s, const uint64_t* addr, uint64_t value);

}  // namespace tcb
