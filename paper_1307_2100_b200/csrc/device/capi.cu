// C-ABI of libtcb200.so (declared in include/tcb.h): context, memory, and the
// argument-checking front of every device operation. Argument errors reproduce
// the reference backend's messages (src/kernels_reference.cpp:12-24) so a
// caller that mapped them to std::invalid_argument sees the same text.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <mutex>
#include <unordered_map>
#include <map>
#include <string>

#include "tcb_internal.cuh"

namespace tcb {

namespace {
struct ThreadCtx {
  int device = -1;  // bound by tcb_init (or lazily to 0)
  ThreadState per[kMaxDevices];
  std::string err;
};
ThreadCtx& ctx() {
  static thread_local ThreadCtx c;
  return c;
}
}  // namespace

ThreadState& state() {
  ThreadCtx& c = ctx();
  return c.per[c.device < 0 ? 0 : c.device];
}

std::string& thread_error() { return ctx().err; }

int set_error(int code, const std::string& msg) {
  ctx().err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  std::string m = std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                  cudaGetErrorString(e) + ")";
  return set_error(e == cudaErrorMemoryAllocation ? TCB_ENOMEM : TCB_ECUDA, m);
}

int num_sms() {
  static int cached[64] = {0};
  int dev = state().device < 0 ? 0 : state().device;
  if (dev < 64 && cached[dev]) return cached[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev < 64) cached[dev] = n;
  return n;
}

int ensure_init() {
  const int dev = ctx().device;
  if (dev >= 0) {
    TCB_CUDA(cudaSetDevice(dev));
    return TCB_OK;
  }
  return tcb_init(0);
}

}  // namespace tcb

namespace tcb {
namespace {
using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned);
struct MemOps {
  WriteValueFn write = nullptr, wait = nullptr;
};
const MemOps& mem_ops() {
  static MemOps ops = [] {
    MemOps o;
    int dev = 0, ok = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&ok, static_cast<cudaDeviceAttr>(CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS),
                           dev);
    if (!ok) return o;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      o.write = reinterpret_cast<WriteValueFn>(f);
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      o.wait = reinterpret_cast<WriteValueFn>(f);
    return o;
  }();
  return ops;
}
}  // namespace

int stream_write_value(cudaStream_t s, uint64_t* addr, uint64_t value) {
  const MemOps& o = mem_ops();
  if (!o.write) return set_error(TCB_EUNSUPPORTED, "64-bit stream memory operations unavailable");
  // default flags: a memory barrier orders the stream's earlier copies first
  const CUresult r = o.write(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr),
                             value, CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return set_error(TCB_ECUDA, "cuStreamWriteValue64 failed");
  return TCB_OK;
}

int stream_wait_value(cudaStream_t s, const uint64_t* addr, uint64_t value) {
  const MemOps& o = mem_ops();
  if (!o.wait) return set_error(TCB_EUNSUPPORTED, "64-bit stream memory operations unavailable");
  const CUresult r = o.wait(reinterpret_cast<CUstream>(s),
                            reinterpret_cast<CUdeviceptr>(const_cast<uint64_t*>(addr)), value,
                            CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return set_error(TCB_ECUDA, "cuStreamWaitValue64 failed");
  return TCB_OK;
}
}  // namespace tcb

using namespace tcb;

#define TCB_TRY_INIT()              \
  do {                              \
    int rc_ = ensure_init();        \
    if (rc_ != TCB_OK) return rc_;  \
  } while (0)

extern "C" {

int tcb_init(int device) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (n == 0) return set_error(TCB_ECUDA, "no CUDA device visible");
  if (device < 0 || device >= n) return set_error(TCB_EINVAL, "tcb_init: device out of range");
  if (device >= kMaxDevices) return set_error(TCB_EUNSUPPORTED, "tcb_init: device index above 15");
  TCB_CUDA(cudaSetDevice(device));
  ctx().device = device;
  ThreadState& st = state();
  if (!st.own_stream) {  // first use of this device by this thread
    TCB_CUDA(cudaStreamCreateWithFlags(&st.own_stream, cudaStreamNonBlocking));
    TCB_CUDA(cudaEventCreate(&st.ev0));
    TCB_CUDA(cudaEventCreate(&st.ev1));
    TCB_CUDA(cudaEventCreateWithFlags(&st.order, cudaEventDisableTiming));
    st.stream = st.own_stream;
    st.device = device;
  }
  return TCB_OK;
}

// Device memory comes from the device's stream-ordered pool with no release
// threshold: freed blocks stay cached for the next allocation (a prepared
// contraction's buffers, a tc::execute call's scratch) instead of going back
// to the driver — cudaMalloc/cudaFree cost milliseconds per call for the
// reference API's allocate-per-evaluation pattern. Semantics stay those of
// cudaMalloc/cudaFree: the block is usable on any stream on return, and a
// free waits for the device first. On exhaustion the pool is trimmed and the
// allocation retried.
static cudaMemPool_t device_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[dev & 63]) {
    cudaMemPool_t pool = nullptr;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return nullptr;
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[dev & 63] = pool;
  }
  return pools[dev & 63];
}

// Exact-size cache of idle device blocks in front of the stream-ordered pool.
// The drop-in tc::execute allocates its operands and result per call; the
// pool did not reliably hand the freed block back (cudaMallocAsync of cfg3's
// 134 MB result took 0.2-7 ms — up to 109 ms — in about half the calls). A
// freed block is idle (tcb_free synchronises the device first, like
// cudaFree), so it can serve the next allocation of the same size on any
// stream at once. Bounded (blocks and bytes per device); flushed back to the
// pool when an allocation fails and by tcb_finalize. The pool itself keeps
// freed memory reserved anyway (release threshold: never).
namespace {
constexpr int kCacheMaxBlocks = 32;
constexpr int64_t kCacheMaxBytes = 64LL << 30;
struct BlockCache {
  std::mutex mu;
  std::unordered_map<void*, int64_t> live[64];        // tcb_alloc'ed blocks -> size
  std::multimap<int64_t, void*> idle[64];             // cached idle blocks by size
  int64_t idle_bytes[64] = {};
};
BlockCache& block_cache() {
  static BlockCache* c = new BlockCache;  // process lifetime (no exit-order issues)
  return *c;
}
// back to the pool: every cached block of the device (stream-ordered free)
void flush_cache(int dev, cudaStream_t stream) {
  BlockCache& c = block_cache();
  std::lock_guard<std::mutex> lock(c.mu);
  for (auto& kv : c.idle[dev]) {
    c.live[dev].erase(kv.second);
    cudaFreeAsync(kv.second, stream);
  }
  c.idle[dev].clear();
  c.idle_bytes[dev] = 0;
}
}  // namespace

int tcb_finalize(void) {
  // releases the calling thread's state on every device it used
  ThreadCtx& c = ctx();
  for (int d = 0; d < kMaxDevices; ++d) {
    ThreadState& st = c.per[d];
    if (st.device < 0) continue;
    cudaSetDevice(d);
    if (st.stream) cudaStreamSynchronize(st.stream);
    if (cudaMemPool_t pool = device_pool()) {  // hand cached blocks back to the driver
      cudaDeviceSynchronize();
      flush_cache(d, st.stream);
      cudaStreamSynchronize(st.stream);
      cudaMemPoolTrimTo(pool, 0);
    }
    if (st.ws) cudaFree(st.ws);
    if (st.counters) cudaFree(st.counters);
    if (st.pace) cudaFree(st.pace);
    if (st.own_stream) cudaStreamDestroy(st.own_stream);
    if (st.ev0) cudaEventDestroy(st.ev0);
    if (st.ev1) cudaEventDestroy(st.ev1);
    if (st.order) cudaEventDestroy(st.order);
    st = ThreadState{};
  }
  c.device = -1;
  return TCB_OK;
}

int tcb_device_count(int* count) {
  if (!count) return set_error(TCB_EINVAL, "tcb_device_count: null pointer");
  *count = 0;
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  return TCB_OK;
}

int tcb_current_device(int* device) {
  if (!device) return set_error(TCB_EINVAL, "tcb_current_device: null pointer");
  *device = ctx().device;
  return TCB_OK;
}

const char* tcb_last_error(void) { return ctx().err.c_str(); }

int tcb_set_stream(void* stream) {
  TCB_TRY_INIT();
  ThreadState& st = state();
  cudaStream_t next = stream ? static_cast<cudaStream_t>(stream) : st.own_stream;
  if (next != st.stream) {
    // The thread's stream-K workspace and tile counters assume stream order:
    // work enqueued from now on waits for what this thread left on the
    // previous stream, so two stream-K GEMMs of one thread never overlap.
    TCB_CUDA(cudaEventRecord(st.order, st.stream));
    TCB_CUDA(cudaStreamWaitEvent(next, st.order, 0));
  }
  st.stream = next;
  st.pdl_ok = false;
  return TCB_OK;
}

int tcb_sync(void) {
  TCB_TRY_INIT();
  TCB_CUDA(cudaStreamSynchronize(state().stream));
  return TCB_OK;
}

int tcb_alloc(void** dptr, int64_t bytes) {
  TCB_TRY_INIT();
  if (!dptr || bytes < 0) return set_error(TCB_EINVAL, "tcb_alloc: bad argument");
  *dptr = nullptr;
  if (bytes == 0) return TCB_OK;
  ThreadState& st = state();
  const int dev = st.device & 63;
  BlockCache& cache = block_cache();
  {
    std::lock_guard<std::mutex> lock(cache.mu);
    auto it = cache.idle[dev].find(bytes);
    if (it != cache.idle[dev].end()) {
      *dptr = it->second;
      cache.idle[dev].erase(it);
      cache.idle_bytes[dev] -= bytes;
      return TCB_OK;
    }
  }
  cudaMemPool_t pool = device_pool();
  cudaError_t e = cudaMallocAsync(dptr, static_cast<size_t>(bytes), st.stream);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    cudaDeviceSynchronize();
    flush_cache(dev, st.stream);
    cudaStreamSynchronize(st.stream);
    if (pool) cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(dptr, static_cast<size_t>(bytes), st.stream);
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
  TCB_CUDA(cudaStreamSynchronize(st.stream));  // usable on every stream, like cudaMalloc
  std::lock_guard<std::mutex> lock(cache.mu);
  cache.live[dev][*dptr] = bytes;
  return TCB_OK;
}

int tcb_free(void* dptr) {
  if (!dptr) return TCB_OK;
  TCB_TRY_INIT();
  TCB_CUDA(cudaDeviceSynchronize());  // cudaFree's implicit synchronisation
  ThreadState& st = state();
  const int dev = st.device & 63;
  BlockCache& cache = block_cache();
  {
    std::lock_guard<std::mutex> lock(cache.mu);
    auto it = cache.live[dev].find(dptr);
    if (it != cache.live[dev].end()) {
      const int64_t bytes = it->second;
      if (static_cast<int>(cache.idle[dev].size()) < kCacheMaxBlocks &&
          cache.idle_bytes[dev] + bytes <= kCacheMaxBytes) {
        cache.idle[dev].emplace(bytes, dptr);  // idle now (device synchronised)
        cache.idle_bytes[dev] += bytes;
        return TCB_OK;
      }
      cache.live[dev].erase(it);
    }
  }
  TCB_CUDA(cudaFreeAsync(dptr, st.stream));
  return TCB_OK;
}

int tcb_memset0(void* dptr, int64_t bytes) {
  TCB_TRY_INIT();
  if (bytes <= 0) return TCB_OK;
  note_stream_op();
  TCB_CUDA(cudaMemsetAsync(dptr, 0, static_cast<size_t>(bytes), state().stream));
  return TCB_OK;
}

static int copy(void* dst, const void* src, int64_t bytes, cudaMemcpyKind kind) {
  TCB_TRY_INIT();
  if (bytes < 0) return set_error(TCB_EINVAL, "copy: negative size");
  if (bytes == 0) return TCB_OK;
  note_stream_op();
  TCB_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), kind, state().stream));
  if (kind == cudaMemcpyDeviceToHost) TCB_CUDA(cudaStreamSynchronize(state().stream));
  return TCB_OK;
}

int tcb_h2d(void* dst, const void* src, int64_t bytes) {
  return copy(dst, src, bytes, cudaMemcpyHostToDevice);
}
int tcb_d2h(void* dst, const void* src, int64_t bytes) {
  return copy(dst, src, bytes, cudaMemcpyDeviceToHost);
}
int tcb_d2d(void* dst, const void* src, int64_t bytes) {
  return copy(dst, src, bytes, cudaMemcpyDeviceToDevice);
}

int tcb_host_register(void* ptr, int64_t bytes) {
  TCB_TRY_INIT();
  if (!ptr || bytes <= 0) return TCB_OK;
  cudaError_t e = cudaHostRegister(ptr, static_cast<size_t>(bytes), cudaHostRegisterDefault);
  if (e == cudaErrorHostMemoryAlreadyRegistered) {
    cudaGetLastError();
    return TCB_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaHostRegister");
  return TCB_OK;
}

int tcb_host_unregister(void* ptr) {
  TCB_TRY_INIT();
  if (!ptr) return TCB_OK;
  cudaError_t e = cudaHostUnregister(ptr);
  if (e == cudaErrorHostMemoryNotRegistered) {
    cudaGetLastError();
    return TCB_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaHostUnregister");
  return TCB_OK;
}

int tcb_stream_create(void** stream) {
  TCB_TRY_INIT();
  if (!stream) return set_error(TCB_EINVAL, "tcb_stream_create: null pointer");
  cudaStream_t s = nullptr;
  TCB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *stream = s;
  return TCB_OK;
}

int tcb_stream_destroy(void* stream) {
  if (!stream) return TCB_OK;
  TCB_TRY_INIT();
  TCB_CUDA(cudaStreamDestroy(static_cast<cudaStream_t>(stream)));
  return TCB_OK;
}

int tcb_event_create(void** event) {
  TCB_TRY_INIT();
  if (!event) return set_error(TCB_EINVAL, "tcb_event_create: null pointer");
  cudaEvent_t e = nullptr;
  TCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  *event = e;
  return TCB_OK;
}

int tcb_event_create_timed(void** event) {
  TCB_TRY_INIT();
  if (!event) return set_error(TCB_EINVAL, "tcb_event_create_timed: null pointer");
  cudaEvent_t e = nullptr;
  TCB_CUDA(cudaEventCreate(&e));
  *event = e;
  return TCB_OK;
}

int tcb_event_destroy(void* event) {
  if (!event) return TCB_OK;
  TCB_TRY_INIT();
  TCB_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(event)));
  return TCB_OK;
}

static cudaStream_t stream_or_current(void* s) {
  return s ? static_cast<cudaStream_t>(s) : state().stream;
}

int tcb_event_sync(void* event) {
  TCB_TRY_INIT();
  if (!event) return set_error(TCB_EINVAL, "tcb_event_sync: null event");
  TCB_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(event)));
  return TCB_OK;
}

int tcb_host_alloc(void** ptr, int64_t bytes) {
  TCB_TRY_INIT();
  if (!ptr || bytes < 0) return set_error(TCB_EINVAL, "tcb_host_alloc: bad argument");
  *ptr = nullptr;
  if (bytes == 0) return TCB_OK;
  TCB_CUDA(cudaHostAlloc(ptr, static_cast<size_t>(bytes), cudaHostAllocPortable));
  return TCB_OK;
}

int tcb_host_free(void* ptr) {
  if (!ptr) return TCB_OK;
  TCB_TRY_INIT();
  TCB_CUDA(cudaFreeHost(ptr));
  return TCB_OK;
}

int tcb_event_record(void* event, void* stream) {
  TCB_TRY_INIT();
  TCB_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(event), stream_or_current(stream)));
  return TCB_OK;
}

int tcb_stream_wait_event(void* stream, void* event) {
  TCB_TRY_INIT();
  note_stream_op(stream_or_current(stream));
  TCB_CUDA(cudaStreamWaitEvent(stream_or_current(stream), static_cast<cudaEvent_t>(event), 0));
  return TCB_OK;
}

int tcb_stream_sync(void* stream) {
  TCB_TRY_INIT();
  TCB_CUDA(cudaStreamSynchronize(stream_or_current(stream)));
  return TCB_OK;
}

void* tcb_current_stream(void) {
  if (ensure_init() != TCB_OK) return nullptr;
  // the caller may enqueue its own work on the stream: the next GEMM must not
  // start before the previous operation ends (no programmatic launch)
  note_stream_op();
  return state().stream;
}

int tcb_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  TCB_TRY_INIT();
  if (bytes < 0) return set_error(TCB_EINVAL, "copy: negative size");
  if (bytes == 0) return TCB_OK;
  note_stream_op(stream_or_current(stream));
  TCB_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault,
                           stream_or_current(stream)));
  return TCB_OK;
}

int tcb_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch,
                       int64_t width, int64_t height, void* stream) {
  TCB_TRY_INIT();
  if (width < 0 || height < 0 || dpitch < width || spitch < width)
    return set_error(TCB_EINVAL, "copy2d: negative size or pitch below width");
  if (width == 0 || height == 0) return TCB_OK;
  note_stream_op(stream_or_current(stream));
  if (height == 1) {
    TCB_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(width), cudaMemcpyDefault,
                             stream_or_current(stream)));
    return TCB_OK;
  }
  TCB_CUDA(cudaMemcpy2DAsync(dst, static_cast<size_t>(dpitch), src, static_cast<size_t>(spitch),
                             static_cast<size_t>(width), static_cast<size_t>(height),
                             cudaMemcpyDefault, stream_or_current(stream)));
  return TCB_OK;
}

int tcb_host_is_pinned(const void* ptr, int* pinned) {
  TCB_TRY_INIT();
  if (!pinned) return set_error(TCB_EINVAL, "tcb_host_is_pinned: null pointer");
  cudaPointerAttributes a{};
  cudaError_t e = cudaPointerGetAttributes(&a, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *pinned = 0;
    return TCB_OK;
  }
  *pinned = a.type == cudaMemoryTypeHost ? 1 : 0;
  return TCB_OK;
}

static int check_desc(const tcb_gemm_desc* d) {
  if (!d) return set_error(TCB_EINVAL, "gemm: null descriptor");
  if (d->m < 0 || d->n < 0 || d->k < 0) return set_error(TCB_EINVAL, "gemm: negative dimension");
  if (d->c_nrow < 1 || d->c_nrow > TCB_MAX_DIMS || d->c_ncol < 1 || d->c_ncol > TCB_MAX_DIMS ||
      d->nbatch < 0 || d->nbatch > TCB_MAX_DIMS)
    return set_error(TCB_EUNSUPPORTED, "gemm: index-group rank outside [1, 6]");
  int64_t pr = 1, pc = 1;
  for (int i = 0; i < d->c_nrow; ++i) pr *= d->c_row_ext[i];
  for (int i = 0; i < d->c_ncol; ++i) pc *= d->c_col_ext[i];
  if (pr != d->m || pc != d->n)
    return set_error(TCB_EINVAL, "gemm: output index groups do not cover m x n");
  for (int i = 0; i < d->nbatch; ++i)
    if (d->bat_ext[i] <= 0) return set_error(TCB_EINVAL, "gemm: batch extent must be positive");
  if (d->g_m != 0 || d->g_n != 0 || d->g_k != 0) {
    if (d->g_m < 1 || d->g_m > TCB_MAX_DIMS || d->g_n < 1 || d->g_n > TCB_MAX_DIMS ||
        d->g_k < 1 || d->g_k > TCB_MAX_DIMS)
      return set_error(TCB_EUNSUPPORTED, "gemm: operand index-group rank outside [1, 6]");
    int64_t pm = 1, pn = 1, pk = 1;
    for (int i = 0; i < d->g_m; ++i) pm *= d->m_ext[i];
    for (int i = 0; i < d->g_n; ++i) pn *= d->n_ext[i];
    for (int i = 0; i < d->g_k; ++i) pk *= d->k_ext[i];
    if (pm != d->m || pn != d->n || pk != d->k)
      return set_error(TCB_EINVAL, "gemm: operand index groups do not cover m, n, k");
    if (d->m < 2 || d->n < 2)
      return set_error(TCB_EUNSUPPORTED, "gemm: operand index groups need m, n >= 2");
  }
  return TCB_OK;
}

int tcb_gemm_check(const tcb_gemm_desc* d) {
  TCB_TRY_INIT();
  const int rc = check_desc(d);
  if (rc != TCB_OK) return rc;
  return check_gemm_groups(*d);
}

int tcb_gemm(const tcb_gemm_desc* d, const double* A, const double* B, double* C) {
  TCB_TRY_INIT();
  int rc = check_desc(d);
  if (rc != TCB_OK) return rc;
  ThreadState& st = state();
  st.last_info = tcb_gemm_info{};
  int64_t batch = 1;
  for (int i = 0; i < d->nbatch; ++i) batch *= d->bat_ext[i];
  if (d->m == 0 || d->n == 0 || batch == 0) return TCB_OK;
  if (d->alpha == 0.0 || d->k == 0) {
    if (d->beta == 1.0) return TCB_OK;
    rc = launch_scale(*d, C);
    st.last_info.launches = 1;
    return rc;
  }
  if (d->n == 1 || d->m == 1) return launch_gemv(*d, A, B, C);
  return launch_gemm(*d, A, B, C);
}

int tcb_stream_write_value(void* stream, uint64_t* addr, uint64_t value) {
  TCB_TRY_INIT();
  if (!addr) return set_error(TCB_EINVAL, "tcb_stream_write_value: null address");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : state().stream;
  note_stream_op(s);
  return stream_write_value(s, addr, value);
}

int tcb_gemm_gated(const tcb_gemm_desc* d, const double* A, const double* B, double* C,
                   const uint64_t* gate, uint64_t value) {
  TCB_TRY_INIT();
  if (!gate) return tcb_gemm(d, A, B, C);
  int rc = check_desc(d);
  if (rc != TCB_OK) return rc;
  ThreadState& st = state();
  int64_t batch = 1;
  for (int i = 0; i < d->nbatch; ++i) batch *= d->bat_ext[i];
  const bool dmma = !(d->m == 0 || d->n == 0 || batch == 0 || d->alpha == 0.0 || d->k == 0 ||
                      d->n == 1 || d->m == 1);
  if (!dmma) {  // paths without a device-side gate: wait in the stream
    note_stream_op();
    rc = stream_wait_value(st.stream, gate, value);
    if (rc != TCB_OK) return rc;
    return tcb_gemm(d, A, B, C);
  }
  st.last_info = tcb_gemm_info{};
  st.gate = reinterpret_cast<const unsigned long long*>(gate);
  st.gate_value = value;
  rc = launch_gemm(*d, A, B, C);
  st.gate = nullptr;
  return rc;
}

int tcb_last_gemm_info(tcb_gemm_info* info) {
  if (!info) return set_error(TCB_EINVAL, "tcb_last_gemm_info: null pointer");
  *info = state().last_info;
  return TCB_OK;
}

// Reference argument checks, src/kernels_reference.cpp:12-24.
static int check_blas(int ta, int tb, int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb,
                      int64_t ldc) {
  if (m < 0 || n < 0 || k < 0) return set_error(TCB_EINVAL, "gemm: negative dimension");
  const int64_t a_rows = ta ? k : m;
  const int64_t b_rows = tb ? n : k;
  if (lda < std::max<int64_t>(1, a_rows)) return set_error(TCB_EINVAL, "gemm: lda below row count");
  if (ldb < std::max<int64_t>(1, b_rows)) return set_error(TCB_EINVAL, "gemm: ldb below row count");
  if (ldc < std::max<int64_t>(1, m)) return set_error(TCB_EINVAL, "gemm: ldc below row count");
  return TCB_OK;
}

static void blas_desc(tcb_gemm_desc* d, int ta, int tb, int64_t m, int64_t n, int64_t k,
                      double alpha, int64_t lda, int64_t ldb, double beta, int64_t ldc) {
  std::memset(d, 0, sizeof *d);
  d->m = m;
  d->n = n;
  d->k = k;
  d->a_sm = ta ? lda : 1;
  d->a_sk = ta ? 1 : lda;
  d->b_sk = tb ? ldb : 1;
  d->b_sn = tb ? 1 : ldb;
  d->c_nrow = d->c_ncol = 1;
  d->c_row_ext[0] = m;
  d->c_row_str[0] = 1;
  d->c_col_ext[0] = n;
  d->c_col_str[0] = ldc;
  d->alpha = alpha;
  d->beta = beta;
}

int tcb_dgemm(int trans_a, int trans_b, int64_t m, int64_t n, int64_t k, double alpha,
              const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
              int64_t ldc) {
  int rc = check_blas(trans_a, trans_b, m, n, k, lda, ldb, ldc);
  if (rc != TCB_OK) return rc;
  tcb_gemm_desc d;
  blas_desc(&d, trans_a, trans_b, m, n, k, alpha, lda, ldb, beta, ldc);
  return tcb_gemm(&d, A, B, C);
}

int tcb_dgemm_strided_batched(int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                              double alpha, const double* A, int64_t lda, int64_t stride_a,
                              const double* B, int64_t ldb, int64_t stride_b, double beta,
                              double* C, int64_t ldc, int64_t stride_c, int64_t batch) {
  int rc = check_blas(trans_a, trans_b, m, n, k, lda, ldb, ldc);
  if (rc != TCB_OK) return rc;
  if (batch < 0) return set_error(TCB_EINVAL, "gemm: negative batch count");
  tcb_gemm_desc d;
  blas_desc(&d, trans_a, trans_b, m, n, k, alpha, lda, ldb, beta, ldc);
  d.nbatch = 1;
  d.bat_ext[0] = batch;
  d.bat_sa[0] = stride_a;
  d.bat_sb[0] = stride_b;
  d.bat_sc[0] = stride_c;
  if (batch == 0) return TCB_OK;
  return tcb_gemm(&d, A, B, C);
}

int tcb_dgemv(int trans, int64_t m, int64_t n, double alpha, const double* A, int64_t lda,
              const double* x, int64_t incx, double beta, double* y, int64_t incy) {
  // Reference checks, src/kernels_reference.cpp:84-86.
  if (m < 0 || n < 0) return set_error(TCB_EINVAL, "gemv: negative dimension");
  if (lda < std::max<int64_t>(1, m)) return set_error(TCB_EINVAL, "gemv: lda below row count");
  tcb_gemm_desc d;
  std::memset(&d, 0, sizeof d);
  // y(len ylen) = op(A) x : as an (ylen x 1) = (ylen x xlen)(xlen x 1) product
  const int64_t ylen = trans ? n : m, xlen = trans ? m : n;
  d.m = ylen;
  d.n = 1;
  d.k = xlen;
  d.a_sm = trans ? lda : 1;
  d.a_sk = trans ? 1 : lda;
  d.b_sk = incx;
  d.b_sn = 1;
  d.c_nrow = d.c_ncol = 1;
  d.c_row_ext[0] = ylen;
  d.c_row_str[0] = incy;
  d.c_col_ext[0] = 1;
  d.c_col_str[0] = 1;
  d.alpha = alpha;
  d.beta = beta;
  return tcb_gemm(&d, A, x, y);
}

int tcb_dger(int64_t m, int64_t n, double alpha, const double* x, int64_t incx, const double* y,
             int64_t incy, double* A, int64_t lda) {
  // Reference checks, src/kernels_reference.cpp:125-127.
  if (m < 0 || n < 0) return set_error(TCB_EINVAL, "ger: negative dimension");
  if (lda < std::max<int64_t>(1, m)) return set_error(TCB_EINVAL, "ger: lda below row count");
  if (alpha == 0.0) return TCB_OK;
  tcb_gemm_desc d;
  std::memset(&d, 0, sizeof d);
  d.m = m;
  d.n = n;
  d.k = 1;
  d.a_sm = incx;
  d.a_sk = 1;
  d.b_sk = 1;
  d.b_sn = incy;
  d.c_nrow = d.c_ncol = 1;
  d.c_row_ext[0] = m;
  d.c_row_str[0] = 1;
  d.c_col_ext[0] = n;
  d.c_col_str[0] = lda;
  d.alpha = alpha;
  d.beta = 1.0;
  return tcb_gemm(&d, x, y, A);
}

int tcb_ddot(int64_t k, const double* x, int64_t incx, const double* y, int64_t incy,
             double* result_host) {
  TCB_TRY_INIT();
  if (!result_host) return set_error(TCB_EINVAL, "dot: null result pointer");
  *result_host = 0.0;
  if (k <= 0) return TCB_OK;
  ThreadState& st = state();
  double* dres = nullptr;
  TCB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dres), 8, st.stream));
  tcb_gemm_desc d;
  std::memset(&d, 0, sizeof d);
  d.m = 1;
  d.n = 1;
  d.k = k;
  d.a_sm = 1;
  d.a_sk = incx;
  d.b_sk = incy;
  d.b_sn = 1;
  d.c_nrow = d.c_ncol = 1;
  d.c_row_ext[0] = d.c_col_ext[0] = 1;
  d.c_row_str[0] = d.c_col_str[0] = 1;
  d.alpha = 1.0;
  d.beta = 0.0;
  int rc = tcb_gemm(&d, x, y, dres);
  if (rc == TCB_OK) {
    note_stream_op();
    cudaError_t e = cudaMemcpyAsync(result_host, dres, 8, cudaMemcpyDeviceToHost, st.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st.stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "dot result copy");
  }
  cudaFreeAsync(dres, st.stream);
  return rc;
}

int tcb_permute(int rank, const int64_t* ext, const int64_t* src_str, const double* src,
                double* dst) {
  TCB_TRY_INIT();
  if (rank < 0 || (rank > 0 && (!ext || !src_str)))
    return set_error(TCB_EINVAL, "permute: bad argument");
  return launch_permute(rank, ext, src_str, src, dst);
}

int tcb_timer_start(void) {
  TCB_TRY_INIT();
  TCB_CUDA(cudaEventRecord(state().ev0, state().stream));
  return TCB_OK;
}

int tcb_timer_stop(float* ms) {
  TCB_TRY_INIT();
  ThreadState& st = state();
  TCB_CUDA(cudaEventRecord(st.ev1, st.stream));
  TCB_CUDA(cudaEventSynchronize(st.ev1));
  float v = 0.f;
  TCB_CUDA(cudaEventElapsedTime(&v, st.ev0, st.ev1));
  if (ms) *ms = v;
  return TCB_OK;
}

int tcb_event_elapsed(void* start, void* stop, float* ms) {
  TCB_TRY_INIT();
  if (!start || !stop || !ms) return set_error(TCB_EINVAL, "tcb_event_elapsed: null argument");
  TCB_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(stop)));
  TCB_CUDA(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start),
                                static_cast<cudaEvent_t>(stop)));
  return TCB_OK;
}

// Synchronous strided copies (the survey's tcb_h2d_2d / tcb_d2h_2d): the
// 2-D copy on the thread's stream, then a wait for it.
int tcb_h2d_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
               int64_t height) {
  const int rc = tcb_memcpy2d_async(dst, dpitch, src, spitch, width, height, nullptr);
  if (rc != TCB_OK) return rc;
  TCB_CUDA(cudaStreamSynchronize(state().stream));
  return TCB_OK;
}
int tcb_d2h_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
               int64_t height) {
  return tcb_h2d_2d(dst, dpitch, src, spitch, width, height);
}

int64_t tcb_launch_count(void) { return state().launches; }
void tcb_reset_launch_count(void) { state().launches = 0; }

}  // extern "C"
