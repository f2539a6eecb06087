// Peer-memory exchange for the K-split partition (BASELINE cfg5),
// fused with the contraction: instead of contracting into a local partial C and
// then reduce-scattering it (NCCL, tcb_reduce_scatter in comm.cu), every rank's
// GEMM epilogue writes each block of its partial C straight into the owning
// rank's receive buffer over NVLink / NVSwitch while the GEMM is still running
// (tile by tile), and the owner then sums its G received slots locally.
//
// Mechanism (CUDA virtual memory management, no NVSHMEM):
//  * tcb_peer_alloc: each rank creates one exportable physical allocation on its
//    own GPU (its receive buffer + flag words) and exports it as a POSIX file
//    descriptor; the host plumbing passes the descriptors between the processes
//    (Unix-socket SCM_RIGHTS, paper_1307_2100_b200/partition.py);
//  * tcb_peer_window: each rank maps ALL ranks' allocations back to back into
//    one reserved virtual range, owner o at window + o * stride. Inside that
//    window the destination of a block of C is an affine function of the block
//    index, so the ordinary GEMM addresses it as one more composite output
//    sub-index (tc::PreparedContraction::run_scattered); no kernel change, and
//    the TMA-store epilogue writes through the peer mappings;
//  * tcb_peer_signal / tcb_peer_reduce: a release-store of the step's epoch into
//    every owner's flag word for this rank, then each owner waits (acquire) for
//    all G flags and sums the slots in rank order 0..G-1 (deterministic).
//
// Replaces no reference code (the reference is single-process CPU code).
#include <cuda.h>

#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "tcb_internal.cuh"

namespace tcb {
namespace {

struct Driver {
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuMemExportToShareableHandle) export_handle = nullptr;
  decltype(&cuMemImportFromShareableHandle) import_handle = nullptr;
  std::string why;
};

const Driver& drv() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    auto sym = [&](auto& fp, const char* name) {
      void* f = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess || !f) {
        if (d.why.empty()) d.why = std::string("driver entry point missing: ") + name;
        return;
      }
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(f);
    };
    sym(d.create, "cuMemCreate");
    sym(d.release, "cuMemRelease");
    sym(d.reserve, "cuMemAddressReserve");
    sym(d.addr_free, "cuMemAddressFree");
    sym(d.map, "cuMemMap");
    sym(d.unmap, "cuMemUnmap");
    sym(d.set_access, "cuMemSetAccess");
    sym(d.granularity, "cuMemGetAllocationGranularity");
    sym(d.export_handle, "cuMemExportToShareableHandle");
    sym(d.import_handle, "cuMemImportFromShareableHandle");
  });
  return d;
}

int cu_fail(CUresult r, const char* what) {
  return set_error(TCB_ECUDA, std::string(what) + " failed (CUresult " + std::to_string(r) + ")");
}

#define TCB_CU(call)                                \
  do {                                              \
    CUresult r_ = (call);                           \
    if (r_ != CUDA_SUCCESS) return cu_fail(r_, #call); \
  } while (0)

#define TCB_DRV_READY()                                              \
  do {                                                               \
    if (!drv().why.empty()) return set_error(TCB_ECUDA, drv().why);  \
  } while (0)

// A mapped range: the reservation, and the (handle, offset, size) pieces in it.
struct Mapping {
  CUdeviceptr base = 0;
  size_t bytes = 0;
  std::vector<CUmemGenericAllocationHandle> handles;
  std::vector<size_t> sizes;
};

std::mutex g_mu;
std::unordered_map<uintptr_t, Mapping> g_maps;  // key: base address

CUmemAllocationProp prop_for(int device) {
  CUmemAllocationProp p = {};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

int release_mapping(Mapping& m) {
  const Driver& d = drv();
  size_t off = 0;
  int rc = TCB_OK;
  for (size_t i = 0; i < m.handles.size(); ++i) {
    if (d.unmap(m.base + off, m.sizes[i]) != CUDA_SUCCESS) rc = TCB_ECUDA;
    if (d.release(m.handles[i]) != CUDA_SUCCESS) rc = TCB_ECUDA;
    off += m.sizes[i];
  }
  if (m.base && d.addr_free(m.base, m.bytes) != CUDA_SUCCESS) rc = TCB_ECUDA;
  return rc == TCB_OK ? TCB_OK : set_error(TCB_ECUDA, "tcb_peer: unmap/release failed");
}

// ------------------------------------------------------------------ kernels

__global__ void peer_signal_kernel(char* window, int64_t stride, int64_t flag_off, int rank,
                                   int world, unsigned long long epoch) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= world) return;
  auto* f = reinterpret_cast<unsigned long long*>(window + o * stride + flag_off) + rank;
  // everything this stream wrote before (the scattered GEMM, an earlier kernel)
  // happens-before this release; the owner's acquire makes it visible there
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(epoch) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// out[i] = sum_{s=0..world-1} slots[s * slot_stride + i], s in order. Every
// block first waits until all `world` flags have reached `epoch`. HBM-bound
// (reads world blocks, writes one): each thread keeps two 16-byte elements x
// four slots of loads in flight before adding them in slot order.
__device__ __forceinline__ void add2(double2& a, const double2 v) {
  a.x += v.x;
  a.y += v.y;
}

__global__ void __launch_bounds__(256) peer_reduce_kernel(
    const double* __restrict__ slots, int world, int64_t count, int64_t slot_stride,
    double* __restrict__ out, const unsigned long long* flags, unsigned long long epoch) {
  if (threadIdx.x < world) {
    const unsigned long long* f = flags + threadIdx.x;
    const unsigned long long t0 = wait_clock_ns();
    while (ld_acquire_sys(f) < epoch) {
      __nanosleep(256);
      if (wait_clock_ns() - t0 > kWaitTrapNs) __trap();  // a peer rank never signalled
    }
  }
  __syncthreads();
  const double2* src = reinterpret_cast<const double2*>(slots);
  const int64_t ss = slot_stride / 2;  // in double2
  const int64_t n2 = count / 2;
  const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n2;
       i += 2 * step) {
    const int64_t j = i + step;
    const bool two = j < n2;
    double2 a = __ldcs(src + i);
    double2 b = two ? __ldcs(src + j) : make_double2(0.0, 0.0);
    int s = 1;
    for (; s + 4 <= world; s += 4) {
      double2 va[4], vb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        va[u] = __ldcs(src + (s + u) * ss + i);
        vb[u] = two ? __ldcs(src + (s + u) * ss + j) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        add2(a, va[u]);
        add2(b, vb[u]);
      }
    }
    for (; s < world; ++s) {
      add2(a, __ldcs(src + s * ss + i));
      if (two) add2(b, __ldcs(src + s * ss + j));
    }
    __stcs(reinterpret_cast<double2*>(out) + i, a);
    if (two) __stcs(reinterpret_cast<double2*>(out) + j, b);
  }
  if (count & 1) {
    const int64_t i = count - 1;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      double acc = slots[i];
      for (int s = 1; s < world; ++s) acc += slots[s * slot_stride + i];
      out[i] = acc;
    }
  }
}

}  // namespace
}  // namespace tcb

using namespace tcb;

extern "C" {

int tcb_peer_granularity(int64_t* bytes) {
  const int rc = ensure_init();
  if (rc != TCB_OK) return rc;
  TCB_DRV_READY();
  if (!bytes) return set_error(TCB_EINVAL, "tcb_peer_granularity: null pointer");
  CUmemAllocationProp p = prop_for(state().device);
  size_t g = 0;
  TCB_CU(drv().granularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  *bytes = static_cast<int64_t>(g);
  return TCB_OK;
}

int tcb_peer_alloc(int64_t bytes, void** dptr, int* fd) {
  const int rc = ensure_init();
  if (rc != TCB_OK) return rc;
  TCB_DRV_READY();
  if (!dptr || !fd) return set_error(TCB_EINVAL, "tcb_peer_alloc: null pointer");
  int64_t g = 0;
  if (tcb_peer_granularity(&g) != TCB_OK) return TCB_ECUDA;
  if (bytes <= 0 || bytes % g)
    return set_error(TCB_EINVAL, "tcb_peer_alloc: size must be a positive multiple of " +
                                     std::to_string(g) + " bytes (tcb_peer_granularity)");
  const Driver& d = drv();
  const int dev = state().device;
  CUmemAllocationProp p = prop_for(dev);
  Mapping m;
  m.bytes = static_cast<size_t>(bytes);
  CUmemGenericAllocationHandle h = 0;
  TCB_CU(d.create(&h, m.bytes, &p, 0));
  m.handles.push_back(h);
  m.sizes.push_back(m.bytes);
  CUresult r = d.reserve(&m.base, m.bytes, static_cast<size_t>(g), 0, 0);
  if (r == CUDA_SUCCESS) r = d.map(m.base, m.bytes, 0, h, 0);
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (r == CUDA_SUCCESS) r = d.set_access(m.base, m.bytes, &acc, 1);
  int shared_fd = -1;
  if (r == CUDA_SUCCESS)
    r = d.export_handle(&shared_fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  if (r != CUDA_SUCCESS) {
    d.release(h);
    if (m.base) d.addr_free(m.base, m.bytes);
    return cu_fail(r, "tcb_peer_alloc (cuMemCreate/Map/SetAccess/Export)");
  }
  TCB_CUDA(cudaMemsetAsync(reinterpret_cast<void*>(m.base), 0, m.bytes, state().stream));
  TCB_CUDA(cudaStreamSynchronize(state().stream));
  note_stream_op();
  *dptr = reinterpret_cast<void*>(m.base);
  *fd = shared_fd;
  std::lock_guard<std::mutex> lk(g_mu);
  g_maps[static_cast<uintptr_t>(m.base)] = std::move(m);
  return TCB_OK;
}

int tcb_peer_window(int n, const int* fds, int64_t stride, void** window) {
  const int rc = ensure_init();
  if (rc != TCB_OK) return rc;
  TCB_DRV_READY();
  if (!fds || !window || n < 1) return set_error(TCB_EINVAL, "tcb_peer_window: bad arguments");
  int64_t g = 0;
  if (tcb_peer_granularity(&g) != TCB_OK) return TCB_ECUDA;
  if (stride <= 0 || stride % g)
    return set_error(TCB_EINVAL, "tcb_peer_window: stride must be a positive multiple of the "
                                 "granularity and equal to every rank's tcb_peer_alloc size");
  const Driver& d = drv();
  Mapping m;
  m.bytes = static_cast<size_t>(stride) * static_cast<size_t>(n);
  TCB_CU(d.reserve(&m.base, m.bytes, static_cast<size_t>(g), 0, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = state().device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (int i = 0; i < n; ++i) {
    CUmemGenericAllocationHandle h = 0;
    CUresult r = d.import_handle(&h, reinterpret_cast<void*>(static_cast<uintptr_t>(fds[i])),
                                 CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    const CUdeviceptr at = m.base + static_cast<size_t>(stride) * i;
    if (r == CUDA_SUCCESS) {
      r = d.map(at, static_cast<size_t>(stride), 0, h, 0);
      if (r != CUDA_SUCCESS) d.release(h);
    }
    if (r != CUDA_SUCCESS) {
      release_mapping(m);
      return cu_fail(r, ("tcb_peer_window: import/map of rank " + std::to_string(i)).c_str());
    }
    m.handles.push_back(h);
    m.sizes.push_back(static_cast<size_t>(stride));
  }
  const CUresult r = d.set_access(m.base, m.bytes, &acc, 1);
  if (r != CUDA_SUCCESS) {
    release_mapping(m);
    return cu_fail(r, "tcb_peer_window: cuMemSetAccess (peer access over NVLink)");
  }
  *window = reinterpret_cast<void*>(m.base);
  std::lock_guard<std::mutex> lk(g_mu);
  g_maps[static_cast<uintptr_t>(m.base)] = std::move(m);
  return TCB_OK;
}

int tcb_peer_free(void* ptr) {
  if (!ptr) return TCB_OK;
  const int rc = ensure_init();
  if (rc != TCB_OK) return rc;
  TCB_DRV_READY();
  Mapping m;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_maps.find(reinterpret_cast<uintptr_t>(ptr));
    if (it == g_maps.end())
      return set_error(TCB_EINVAL, "tcb_peer_free: not a tcb_peer_alloc/tcb_peer_window address");
    m = std::move(it->second);
    g_maps.erase(it);
  }
  TCB_CUDA(cudaDeviceSynchronize());
  return release_mapping(m);
}

int tcb_peer_signal(void* window, int64_t stride, int64_t flag_off, int rank, int world,
                    uint64_t epoch) {
  const int rc = ensure_init();
  if (rc != TCB_OK) return rc;
  if (!window || world < 1 || rank < 0 || rank >= world || flag_off < 0 || flag_off % 8 ||
      flag_off + 8 * world > stride)
    return set_error(TCB_EINVAL, "tcb_peer_signal: bad arguments");
  peer_signal_kernel<<<1, 32 * ((world + 31) / 32), 0, state().stream>>>(
      static_cast<char*>(window), stride, flag_off, rank, world,
      static_cast<unsigned long long>(epoch));
  TCB_LAUNCHED();
  return TCB_OK;
}

int tcb_peer_reduce(const double* slots, int world, int64_t count, int64_t slot_stride,
                    double* out, const uint64_t* flags, uint64_t epoch) {
  const int rc = ensure_init();
  if (rc != TCB_OK) return rc;
  if (!slots || !out || !flags || world < 1 || world > 256 || count < 0 ||
      slot_stride < count || (reinterpret_cast<uintptr_t>(slots) & 15) ||
      (reinterpret_cast<uintptr_t>(out) & 15) || (slot_stride & 1))
    return set_error(TCB_EINVAL,
                     "tcb_peer_reduce: bad arguments (16-byte aligned slots/out, even slot "
                     "stride >= count, 1 <= world <= 256)");
  const int64_t n2 = count / 2;
  const int64_t per = 256LL * 2;  // elements (double2) per block at 2 per thread
  int64_t blocks = (n2 + per - 1) / per;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  peer_reduce_kernel<<<static_cast<unsigned>(blocks), 256, 0, state().stream>>>(
      slots, world, count, slot_stride, out, reinterpret_cast<const unsigned long long*>(flags),
      static_cast<unsigned long long>(epoch));
  TCB_LAUNCHED();
  return TCB_OK;
}

}  // extern "C"
