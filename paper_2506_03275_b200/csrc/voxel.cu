// voxel.cu — voxel token reorder (voxel_order / reverse_voxel_order,
// voxel.cpp:44-102) as a row gather / scatter.
//
// The permutation (voxel.cpp:18-42) is recomputed arithmetically per row, so
// no index array is read from HBM: the kernel moves exactly 2*B*N*row_bytes.
// One warp per row, 16-byte vector accesses when rows are 16 B multiples
// (bf16 D=3072 -> 384 x 16 B per row), byte copies otherwise.  Bit-exact in
// every dtype.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace csd {
namespace dev {

struct VoxelGeom {
    int64_t t, h, w, vt, vh, vw;
};

// new position -> original raster position (voxel.cpp:27-38)
__device__ __forceinline__ int64_t voxel_src(int64_t pos, const VoxelGeom& g) {
    const int64_t vol = g.vt * g.vh * g.vw;
    const int64_t vid = pos / vol, in = pos % vol;
    const int64_t nwc = g.w / g.vw, nhc = g.h / g.vh;
    const int64_t tc = vid / (nhc * nwc), hc = (vid / nwc) % nhc, wc = vid % nwc;
    const int64_t it = in / (g.vh * g.vw), ih = (in / g.vw) % g.vh, iw = in % g.vw;
    return ((tc * g.vt + it) * g.h + hc * g.vh + ih) * g.w + wc * g.vw + iw;
}

template <bool kVec16>
__global__ void k_voxel_reorder(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                int64_t rows_total, int64_t n, int64_t row_bytes, VoxelGeom g,
                                int inverse) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= rows_total) return;
    const int64_t b = warp / n, pos = warp % n;
    const int64_t orig = voxel_src(pos, g);
    const int64_t in_row = b * n + (inverse ? pos : orig);
    const int64_t out_row = b * n + (inverse ? orig : pos);
    const uint8_t* s = src + in_row * row_bytes;
    uint8_t* d = dst + out_row * row_bytes;
    if (kVec16) {
        const uint4* s4 = reinterpret_cast<const uint4*>(s);
        uint4* d4 = reinterpret_cast<uint4*>(d);
        const int64_t nv = row_bytes / 16;
        for (int64_t i = lane; i < nv; i += 32) d4[i] = __ldg(s4 + i);
    } else {
        for (int64_t i = lane; i < row_bytes; i += 32) d[i] = s[i];
    }
}

cudaError_t voxel_reorder(const void* src, void* dst, int64_t batch, int64_t t, int64_t h,
                          int64_t w, int64_t vt, int64_t vh, int64_t vw, int64_t row_bytes,
                          int inverse, cudaStream_t s) {
    const int64_t n = t * h * w;
    const int64_t rows = batch * n;
    if (rows == 0) return cudaSuccess;
    VoxelGeom g{t, h, w, vt, vh, vw};
    const int threads = 256;
    const unsigned blocks = (unsigned)((rows * 32 + threads - 1) / threads);
    const bool vec = (row_bytes % 16 == 0) && (((uintptr_t)src | (uintptr_t)dst) % 16 == 0);
    if (vec)
        k_voxel_reorder<true><<<blocks, threads, 0, s>>>((const uint8_t*)src, (uint8_t*)dst, rows,
                                                         n, row_bytes, g, inverse);
    else
        k_voxel_reorder<false><<<blocks, threads, 0, s>>>((const uint8_t*)src, (uint8_t*)dst,
                                                          rows, n, row_bytes, g, inverse);
    return cudaGetLastError();
}

}  // namespace dev
}  // namespace csd
