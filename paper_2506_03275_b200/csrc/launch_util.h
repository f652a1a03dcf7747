// launch_util.h — host-side launch helpers shared by the kernel translation units.
//
// Kernel attributes (max dynamic shared memory) are per DEVICE: a process-wide "done" flag
// set on the first device would leave every other device's launches above 48 KB failing
// with invalid-argument.  These helpers key the attribute and the SM count on
// (kernel, current device), thread-safely.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
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

// Programmatic dependent launch for the block-step kernels (common.cuh pdl_wait /
// pdl_trigger).  Measured on the FLUX block (r02, CUPTI timeline of graph replays): with
// every kernel behind its predecessor (CSD_PDL=2) the kernels start 12-40 us early but the
// sparse step ends at the same time (425 vs 428 us) -- every kernel's main work depends on
// its predecessor's output and the persistent grids take statically assigned work, so only
// prologues overlap; with the attention kernels alone (CSD_PDL=1: their barrier / TMEM
// setup and dead-warp code warm-up overlap the Q/K/V GEMM's tail) the sparse step measured
// 409.2 -> 405.9 us on one box and 413.4 -> 414.9 us on another: within noise, so it stays
// opt-in (default 0).
// CSD_PDL=1: only the launches that profit (the attention kernels behind the Q/K/V GEMM:
// their code warm-up and barrier / TMEM setup overlap the GEMM's tail); CSD_PDL=2: every
// block-step kernel.
inline int pdl_mode() {
    static const int m = [] {
        const char* e = std::getenv("CSD_PDL");
        return e != nullptr ? std::atoi(e) : 0;
    }();
    return m;
}
inline bool pdl_enabled(int level = 2) { return pdl_mode() >= level; }

// cudaLaunchKernelEx with the programmatic-serialization attribute (when enabled) and an
// optional cluster shape (cluster_x > 1).  Every kernel launched through here calls
// pdl_wait() before its first global-memory access.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex_pdl(int pdl_level, void (*kern)(KArgs...), dim3 grid, dim3 block,
                                 size_t smem, cudaStream_t s, unsigned cluster_x, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl_enabled(pdl_level)) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cluster_x > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = cluster_x;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t s, unsigned cluster_x, Args&&... args) {
    return launch_ex_pdl(2, kern, grid, block, smem, s, cluster_x, std::forward<Args>(args)...);
}

}  // namespace dev
}  // namespace csd
