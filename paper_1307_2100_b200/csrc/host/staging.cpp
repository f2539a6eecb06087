// Pageable host <-> device transfers through pinned bounce buffers.
//
// The reference API hands the engine std::vector storage (include/tc/
// tensor.hpp:58): pageable memory, which the driver copies through its own
// small staging path at a few GB/s. Here large copies are cut into 16 MB
// chunks that cycle through three page-locked buffers: worker threads copy
// chunk i into (or out of) a buffer while the DMA engine moves chunk i-1, so
// a transfer runs at the rate of the slower of the parallel host copy and
// PCIe instead of the serial driver path. Pinned sources/destinations and
// small copies go straight to the DMA engine.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "staging.hpp"
#include "tcb.h"

namespace tc {
namespace {

void check_tcb(int rc, const char* what) {
  if (rc != TCB_OK) throw std::runtime_error(std::string(what) + ": " + tcb_last_error());
}

// A fixed set of worker threads running one parallel copy at a time.
class CopyPool {
 public:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned n = std::min(8u, std::max(1u, hw / 2));
    for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  // dst[0..n) = src[0..n), split over the workers and the calling thread
  void copy(void* dst, const void* src, std::size_t n) {
    std::lock_guard<std::mutex> serial(call_mu_);  // one parallel copy at a time
    const std::size_t parts = workers_.size() + 1;
    const std::size_t piece = (n + parts - 1) / parts;
    {
      std::lock_guard<std::mutex> lk(mu_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      n_ = n;
      piece_ = piece;
      pending_ = workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    const std::size_t lo = std::min(n, workers_.size() * piece);  // caller's own piece: the last
    std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, n - lo);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void loop(unsigned idx) {
    std::size_t seen = 0;
    for (;;) {
      char* dst;
      const char* src;
      std::size_t n, piece;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        dst = dst_;
        src = src_;
        n = n_;
        piece = piece_;
      }
      const std::size_t lo = std::min(n, idx * piece), hi = std::min(n, lo + piece);
      if (hi > lo) std::memcpy(dst + lo, src + lo, hi - lo);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_.notify_all();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_;
  bool stop_ = false;
  std::size_t gen_ = 0, pending_ = 0;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  std::size_t n_ = 0, piece_ = 0;
};

constexpr std::int64_t kChunk = 16LL << 20;
constexpr int kBuffers = 3;
constexpr std::int64_t kDirect = 4LL << 20;  // below this the driver's copy is fine

// Bounce buffers and their "free again" events.
struct Bounce {
  void* buf[kBuffers] = {};
  void* ev[kBuffers] = {};
  ~Bounce() {
    for (int i = 0; i < kBuffers; ++i) {
      if (ev[i]) tcb_event_sync(ev[i]), tcb_event_destroy(ev[i]);
      tcb_host_free(buf[i]);
    }
  }
  void ensure() {
    for (int i = 0; i < kBuffers; ++i) {
      if (!buf[i]) check_tcb(tcb_host_alloc(&buf[i], kChunk), "pinned staging buffer");
      if (!ev[i]) check_tcb(tcb_event_create(&ev[i]), "staging event");
    }
  }
};

CopyPool& pool() {
  static CopyPool p;
  return p;
}
// one set per (thread, device): the events belong to the device they were
// created on, and a thread may alternate between devices
Bounce& bounce() {
  thread_local Bounce b[16];
  int dev = 0;
  tcb_current_device(&dev);
  Bounce& mine = b[dev < 0 ? 0 : dev & 15];
  mine.ensure();
  return mine;
}

bool pinned(const void* p) {
  int is = 0;
  tcb_host_is_pinned(p, &is);
  return is != 0;
}

}  // namespace

void host_to_device(void* dev, const void* host, std::int64_t bytes, void* stream) {
  if (bytes <= 0) return;
  if (bytes < kDirect || pinned(host)) {
    check_tcb(tcb_memcpy_async(dev, host, bytes, stream), "upload");
    if (!pinned(host)) check_tcb(tcb_stream_sync(stream), "upload");
    return;
  }
  Bounce& b = bounce();
  const std::int64_t n = (bytes + kChunk - 1) / kChunk;
  for (std::int64_t i = 0; i < n; ++i) {
    const int k = static_cast<int>(i % kBuffers);
    const std::int64_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    check_tcb(tcb_event_sync(b.ev[k]), "staging");  // buffer k's previous upload has left
    pool().copy(b.buf[k], static_cast<const char*>(host) + off, static_cast<std::size_t>(len));
    check_tcb(tcb_memcpy_async(static_cast<char*>(dev) + off, b.buf[k], len, stream), "upload");
    check_tcb(tcb_event_record(b.ev[k], stream), "staging");
  }
  // the caller's memory may change once this returns; the bounce buffers
  // carry the data, so only their reuse has to wait (next call)
}

void device_to_host(void* host, const void* dev, std::int64_t bytes, void* stream) {
  if (bytes <= 0) return;
  if (bytes < kDirect || pinned(host)) {
    check_tcb(tcb_memcpy_async(host, dev, bytes, stream), "download");
    check_tcb(tcb_stream_sync(stream), "download");
    return;
  }
  Bounce& b = bounce();
  const std::int64_t n = (bytes + kChunk - 1) / kChunk;
  auto issue = [&](std::int64_t i) {
    const int k = static_cast<int>(i % kBuffers);
    const std::int64_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    check_tcb(tcb_memcpy_async(b.buf[k], static_cast<const char*>(dev) + off, len, stream),
              "download");
    check_tcb(tcb_event_record(b.ev[k], stream), "staging");
  };
  for (std::int64_t i = 0; i < std::min<std::int64_t>(n, kBuffers); ++i) issue(i);
  for (std::int64_t i = 0; i < n; ++i) {
    const int k = static_cast<int>(i % kBuffers);
    const std::int64_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    check_tcb(tcb_event_sync(b.ev[k]), "staging");  // chunk i landed in buffer k
    pool().copy(static_cast<char*>(host) + off, b.buf[k], static_cast<std::size_t>(len));
    if (i + kBuffers < n) issue(i + kBuffers);
  }
}

}  // namespace tc
