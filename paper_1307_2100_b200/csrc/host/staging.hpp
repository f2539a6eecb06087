// Pageable-aware host <-> device copies (staging.cpp). Host C++ only.
#pragma once
#include <cstdint>

namespace tc {
// Upload `bytes` from host memory to device memory on `stream` (null: the
// thread's current one). Large pageable sources go through pinned bounce
// buffers with a parallel host copy; the call returns once the source may be
// reused (the device copy completes in stream order).
void host_to_device(void* dev, const void* host, std::int64_t bytes, void* stream);
// Download `bytes` into host memory; returns when the data is on the host.
void device_to_host(void* host, const void* dev, std::int64_t bytes, void* stream);
}  // namespace tc
