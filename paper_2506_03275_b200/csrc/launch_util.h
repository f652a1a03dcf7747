// launch_util.h — host-side launch helpers shared by the kernel translation units.
//
// Kernel attributes (max dynamic shared memory) are per DEVICE: a process-wide "done" flag
// set on the first device would leave every other device's launches above 48 KB failing
// with invalid-argument.  These helpers key the attribute and the SM count on
// (kernel, current device), thread-safely.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <utility>

namespace csd {
namespace dev {

inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

// Set cudaFuncAttributeMaxDynamicSharedMemorySize >= bytes for `fn` on the current device
// (once per (kernel, device, size)).
inline cudaError_t ensure_smem_attr(const void* fn, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> done;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(fn, dev);
    auto it = done.find(key);
    if (it != done.end() && it->second >= bytes) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done[key] = bytes;
    return e;
}
template <typename K>
inline cudaError_t ensure_smem_attr(K* fn, int bytes) {
    return ensure_smem_attr(reinterpret_cast<const void*>(fn), bytes);
}

// SM count of the current device (cached per device).
inline int sm_count() {
    static std::mutex mu;
    static std::map<int, int> cache;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
        n = 148;
    cache[dev] = n;
    return n;
}

}  // namespace dev
}  // namespace csd
