// topk.cu — exact per-row top-k (select_top_k, sparse_index.cpp:64-96) and
// on-device SparseIndexSet::validate (sparse_index.cpp:27-62).
//
// Order contract: descending score, lower index first on equal scores; +0.0
// and -0.0 compare equal (the reference comparator uses `!=` / `>`).  Each
// element maps to a unique 64-bit composite  (ord(score) << 32) | ~index,
// whose descending order IS the reference order, so the k largest composites
// are the answer.  Per row (one CTA):
//   1. 4-pass 8-bit radix select on ord() -> threshold T, G = #{ord > T};
//   2. collect all ord > T plus the (k - G) lowest-index ord == T
//      (block-wide ordered scan, so ties resolve by index);
//   3. bitonic sort of the k composites in shared memory.
// The row is staged in shared memory when it fits (FLUX: 4608 fp32 = 18 KB),
// otherwise re-read from L2 on each pass (Hunyuan rows: 118272 fp32).
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace csd {
namespace dev {

constexpr int kTopkThreads = 512;
constexpr int kTopkWarps = kTopkThreads / 32;
constexpr int64_t kTopkMaxSortK = 16384;         // 128 KB of u64 composites
constexpr int64_t kTopkMaxSmemRow = 16 * 1024;  // fp32 elements staged in smem

__device__ __forceinline__ uint32_t ord_key(float x) {
    uint32_t u = __float_as_uint(x);
    if ((u << 1) == 0) u = 0;  // -0.0 == +0.0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void __launch_bounds__(kTopkThreads)
k_topk_rows(const float* __restrict__ scores, int64_t m, int64_t k, int32_t* __restrict__ idx_out,
            int32_t* __restrict__ counts, int stage_row, int sort_pow2) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* sel = reinterpret_cast<uint64_t*>(smem);                 // [sort_pow2]
    float* srow = reinterpret_cast<float*>(smem + sizeof(uint64_t) * sort_pow2);
    __shared__ uint32_t hist[256];
    __shared__ uint32_t warp_tot[kTopkWarps];
    __shared__ uint32_t s_prefix, s_kleft, s_total, s_gt;

    const int64_t row = blockIdx.x;
    const float* src = scores + row * m;
    const int tid = threadIdx.x;
    if (stage_row) {
        for (int64_t j = tid; j < m; j += kTopkThreads) srow[j] = src[j];
        src = srow;
    }
    if (tid == 0) { s_prefix = 0; s_kleft = (uint32_t)k; s_gt = 0; }
    __syncthreads();

    uint32_t mask = 0;
    // per-warp private histograms: nearby scores share their top digits, so a single
    // shared histogram serialises thousands of same-address atomics
    __shared__ uint32_t whist[kTopkWarps][256];
    const int warp_id = tid >> 5;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = tid; i < kTopkWarps * 256; i += kTopkThreads) (&whist[0][0])[i] = 0;
        __syncthreads();
        const uint32_t prefix = s_prefix;
        uint32_t* wh = whist[warp_id];
        for (int64_t j = tid; j < m; j += kTopkThreads) {
            const uint32_t o = ord_key(src[j]);
            if ((o & mask) == prefix) atomicAdd(&wh[(o >> shift) & 0xffu], 1u);
        }
        __syncthreads();
        for (int i = tid; i < 256; i += kTopkThreads) {
            uint32_t acc = 0;
#pragma unroll
            for (int w = 0; w < kTopkWarps; ++w) acc += whist[w][i];
            hist[i] = acc;
        }
        __syncthreads();
        if (tid < 32) {
            // lane l owns descending digits d = 8l..8l+7  (bin = 255 - d)
            uint32_t c[8], tot = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) { c[i] = hist[255 - (8 * tid + i)]; tot += c[i]; }
            uint32_t incl = tot;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += t;
            }
            uint32_t run = incl - tot;  // elements in higher digits
            const uint32_t need = s_kleft;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (run < need && run + c[i] >= need) {
                    s_prefix = prefix | ((uint32_t)(255 - (8 * tid + i)) << shift);
                    s_kleft = need - run;
                }
                run += c[i];
            }
        }
        mask |= 0xffu << shift;
        __syncthreads();
    }
    const uint32_t T = s_prefix;
    const uint32_t need_eq = s_kleft;           // ties to take, lowest index first
    const uint32_t G = (uint32_t)k - need_eq;   // strictly greater

    // collect: warp w owns the contiguous segment [w*seg, (w+1)*seg); one counting pass,
    // one block scan of the per-warp tie counts (index order = warp order), one write pass
    const int lane = tid & 31;
    const int64_t seg = ((m + kTopkWarps * 32 - 1) / (kTopkWarps * 32)) * 32;
    const int64_t s0 = warp_id * seg, s1 = min(m, s0 + seg);
    uint32_t n_eq = 0;
    for (int64_t j0 = s0; j0 < s1; j0 += 32) {
        const int64_t j = j0 + lane;
        n_eq += __popc(__ballot_sync(0xffffffffu, j < s1 && ord_key(src[j]) == T));
    }
    if (lane == 0) warp_tot[warp_id] = n_eq;
    __syncthreads();
    if (tid < 32) {
        const uint32_t v = tid < kTopkWarps ? warp_tot[tid] : 0u;
        uint32_t incl = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (tid >= o) incl += t;
        }
        if (tid < kTopkWarps) warp_tot[tid] = incl - v;  // exclusive tie offset per warp
    }
    __syncthreads();
    uint32_t eq_run = warp_tot[warp_id];
    for (int64_t j0 = s0; j0 < s1; j0 += 32) {
        const int64_t j = j0 + lane;
        uint32_t o = 0;
        if (j < s1) o = ord_key(src[j]);
        const bool gt = j < s1 && o > T, eq = j < s1 && o == T;
        const uint64_t comp = ((uint64_t)o << 32) | (uint32_t)~(uint32_t)j;
        const uint32_t gb = __ballot_sync(0xffffffffu, gt);
        uint32_t gbase = 0;
        if (lane == 0 && gb) gbase = atomicAdd(&s_gt, (uint32_t)__popc(gb));
        gbase = __shfl_sync(0xffffffffu, gbase, 0);
        if (gt) sel[gbase + __popc(gb & ((1u << lane) - 1u))] = comp;
        const uint32_t eb = __ballot_sync(0xffffffffu, eq);
        const uint32_t r = eq_run + __popc(eb & ((1u << lane) - 1u));
        if (eq && r < need_eq) sel[G + r] = comp;
        eq_run += __popc(eb);
    }
    __syncthreads();
    int32_t* dst = idx_out + row * k;
    if (k <= 2048) {
        // all composites are distinct: output slot = number of selected composites above it
        for (int i = tid; i < k; i += kTopkThreads) {
            const uint64_t c = sel[i];
            int rank = 0;
            for (int q = 0; q < k; ++q) rank += sel[q] > c;
            dst[rank] = (int32_t)(~(uint32_t)c);
        }
        if (tid == 0 && counts) counts[row] = (int32_t)k;
        return;
    }
    for (int i = (int)k + tid; i < sort_pow2; i += kTopkThreads) sel[i] = 0ull;
    __syncthreads();
    // bitonic sort, descending
    for (int size = 2; size <= sort_pow2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < sort_pow2; i += kTopkThreads) {
                const int partner = i ^ stride;
                if (partner > i) {
                    const bool desc = (i & size) == 0;
                    const uint64_t a = sel[i], b = sel[partner];
                    if (desc ? (a < b) : (a > b)) { sel[i] = b; sel[partner] = a; }
                }
            }
            __syncthreads();
        }
    }
    for (int i = tid; i < k; i += kTopkThreads) dst[i] = (int32_t)(~(uint32_t)sel[i]);
    if (tid == 0 && counts) counts[row] = (int32_t)k;
}

// Fallback for k beyond the shared-memory sort: composites staged in global
// memory, output position = number of selected composites larger than it.
__global__ void k_topk_collect_global(const float* __restrict__ scores, int64_t m, int64_t k,
                                      uint64_t* __restrict__ ws) {
    // single pass per row: select via full ranking is O(m^2); used only for
    // huge k where rows are few.  Rank each element among the row.
    const int64_t row = blockIdx.y;
    const float* src = scores + row * m;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t cj = ((uint64_t)ord_key(src[j]) << 32) | (uint32_t)~(uint32_t)j;
        int64_t rank = 0;
        for (int64_t t = 0; t < m; ++t) {
            const uint64_t ct = ((uint64_t)ord_key(src[t]) << 32) | (uint32_t)~(uint32_t)t;
            rank += ct > cj;
        }
        if (rank < k) ws[row * k + rank] = cj;
    }
}

__global__ void k_topk_emit_global(const uint64_t* ws, int64_t rows, int64_t k, int32_t* idx,
                                   int32_t* counts) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < rows * k) idx[i] = (int32_t)(~(uint32_t)ws[i]);
    if (i < rows && counts) counts[i] = (int32_t)k;
}

int64_t topk_max_k() { return kTopkMaxSortK; }

cudaError_t topk_rows(const float* scores, int64_t rows, int64_t m, int64_t k, int32_t* idx,
                      int32_t* counts, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    if (k > kTopkMaxSortK) return cudaErrorNotSupported;  // caller uses topk_rows_global
    int p2 = 1;
    while (p2 < k) p2 <<= 1;
    const int stage = m <= kTopkMaxSmemRow ? 1 : 0;
    const size_t smem = sizeof(uint64_t) * p2 + (stage ? sizeof(float) * m : 0);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_topk_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 196 * 1024);
        attr_set = true;
    }
    k_topk_rows<<<(unsigned)rows, kTopkThreads, smem, s>>>(scores, m, k, idx, counts, stage, p2);
    return cudaGetLastError();
}

cudaError_t topk_rows_global(const float* scores, int64_t rows, int64_t m, int64_t k,
                             int32_t* idx, int32_t* counts, uint64_t* ws, cudaStream_t s) {
    dim3 g((unsigned)((m + 255) / 256), (unsigned)rows);
    k_topk_collect_global<<<g, 256, 0, s>>>(scores, m, k, ws);
    k_topk_emit_global<<<(unsigned)((rows * k + 255) / 256), 256, 0, s>>>(ws, rows, k, idx, counts);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// SparseIndexSet::validate: counts in [0, k_max], ids in [0, domain), unique
// within a row (shared-memory bitmap per row).
__global__ void k_validate(const int32_t* idx, const int32_t* counts, int64_t k_max,
                           int64_t domain, uint32_t* flags) {
    extern __shared__ uint32_t bits[];
    const int64_t row = blockIdx.x;
    const int64_t words = (domain + 31) / 32;
    for (int64_t i = threadIdx.x; i < words; i += blockDim.x) bits[i] = 0;
    __syncthreads();
    const int32_t cnt = counts[row];
    if (cnt < 0 || cnt > k_max) {
        if (threadIdx.x == 0) raise_flag(flags, kFlagCountRange);
        return;
    }
    const int32_t* ids = idx + row * k_max;
    for (int32_t j = threadIdx.x; j < cnt; j += blockDim.x) {
        const int32_t v = ids[j];
        if (v < 0 || v >= domain) { raise_flag(flags, kFlagIndexRange); continue; }
        const uint32_t old = atomicOr(&bits[v >> 5], 1u << (v & 31));
        if (old & (1u << (v & 31))) raise_flag(flags, kFlagIndexDup);
    }
}

cudaError_t validate_index_set(const int32_t* idx, const int32_t* counts, int64_t rows,
                               int64_t k_max, int64_t domain, uint32_t* flags, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    const size_t smem = sizeof(uint32_t) * (size_t)((domain + 31) / 32);
    if (smem > 200 * 1024) return cudaErrorNotSupported;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_validate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    k_validate<<<(unsigned)rows, 256, smem, s>>>(idx, counts, k_max, domain, flags);
    return cudaGetLastError();
}

}  // namespace dev
}  // namespace csd
