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
#include "launch_util.h"
#include "tc_common.cuh"

namespace csd {
namespace dev {

// Debug timeline (scripts/topk_micro.py --trace): CTA 0 stamps clock64() per phase.
__device__ uint64_t* g_topk_trace = nullptr;
#define TOPK_TRACE(slot)                                                                  \
    do {                                                                                  \
        if (blockIdx.x == 0 && threadIdx.x == 0) { /* one thread pays the pointer load */ \
            uint64_t* tr_ = g_topk_trace;                                                 \
            if (tr_ != nullptr) tr_[slot] = clock64();                                    \
        }                                                                                 \
    } while (0)

constexpr int kTopkThreads = 512;
constexpr int kTopkWarps = kTopkThreads / 32;
constexpr int64_t kTopkMaxSortK = 16384;         // 128 KB of u64 composites
constexpr int64_t kTopkMaxSmemRow = 16 * 1024;  // fp32 elements staged in smem

__device__ __forceinline__ uint32_t smem_u32_generic(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t ord_key(float x) {
    uint32_t u = __float_as_uint(x);
    if ((u << 1) == 0) u = 0;  // -0.0 == +0.0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Bitonic sort (descending) of P = sort_pow2 64-bit keys in smem.  Strides >= 64 run over
// smem with a block barrier per step; each run of strides 32..1 runs in registers: a warp
// owns 64-element segments (element lane and 32 + lane), stride 32 is an in-thread swap and
// strides 16..1 are shuffles.
__device__ __forceinline__ void cmp_swap_desc(uint64_t& a, uint64_t& b, bool desc) {
    if (desc ? (a < b) : (a > b)) {
        const uint64_t t = a;
        a = b;
        b = t;
    }
}
__device__ void bitonic_sort_desc(uint64_t* sel, int P) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int size = 2; size <= P; size <<= 1) {
        for (int j = size >> 1; j >= 64; j >>= 1) {
            for (int i = tid; i < P; i += kTopkThreads) {
                const int q = i ^ j;
                if (q > i) {
                    uint64_t a = sel[i], b = sel[q];
                    cmp_swap_desc(a, b, (i & size) == 0);
                    sel[i] = a;
                    sel[q] = b;
                }
            }
            __syncthreads();
        }
        // strides min(size/2, 32) .. 1 in registers, one 64-element segment per warp pass
        for (int seg = warp * 64; seg < P; seg += kTopkWarps * 64) {
            uint64_t r0 = sel[seg + lane], r1 = sel[seg + 32 + lane];
            const int i0 = seg + lane, i1 = seg + 32 + lane;
            for (int j = min(size >> 1, 32); j >= 1; j >>= 1) {
                if (j == 32) {
                    cmp_swap_desc(r0, r1, (i0 & size) == 0);  // partners i0, i0 + 32
                } else {
                    // partner lane^j holds element i^j in the same register
                    const bool lower = (lane & j) == 0;
                    const uint64_t p0 = __shfl_xor_sync(0xffffffffu, r0, j);
                    const uint64_t p1 = __shfl_xor_sync(0xffffffffu, r1, j);
                    const bool d0 = (i0 & size) == 0, d1 = (i1 & size) == 0;
                    // the lower index keeps the larger key when descending
                    const bool take0 = lower ? (d0 ? p0 > r0 : p0 < r0) : (d0 ? p0 < r0 : p0 > r0);
                    const bool take1 = lower ? (d1 ? p1 > r1 : p1 < r1) : (d1 ? p1 < r1 : p1 > r1);
                    r0 = take0 ? p0 : r0;
                    r1 = take1 ? p1 : r1;
                }
            }
            sel[seg + lane] = r0;
            sel[seg + 32 + lane] = r1;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kTopkThreads)
k_topk_rows(const float* __restrict__ scores, int64_t m, int64_t k, int32_t* __restrict__ idx_out,
            int32_t* __restrict__ counts, int stage_row, int sort_pow2, int sorted) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* sel = reinterpret_cast<uint64_t*>(smem);                         // [sort_pow2]
    uint32_t* keys = reinterpret_cast<uint32_t*>(smem + sizeof(uint64_t) * sort_pow2);  // [m]
    __shared__ uint32_t hist[256];
    __shared__ uint32_t warp_tot[2][kTopkWarps];
    __shared__ uint32_t warp_red[2][kTopkWarps];
    __shared__ uint32_t s_prefix, s_kleft;
    pdl_wait();
    if (threadIdx.x == 0) pdl_trigger();

    const int64_t row = blockIdx.x;
    const float* src = scores + row * m;
    const int tid = threadIdx.x, lane = tid & 31, warp_id = tid >> 5;
    TOPK_TRACE(0);
    // ord keys (staged when the row fits) and their common leading bits (AND / OR reduce)
    uint32_t kand = 0xffffffffu, kor = 0u;
    for (int64_t j = tid; j < m; j += kTopkThreads) {
        const uint32_t o = ord_key(src[j]);
        if (stage_row) keys[j] = o;
        kand &= o;
        kor |= o;
    }
    kand = __reduce_and_sync(0xffffffffu, kand);
    kor = __reduce_or_sync(0xffffffffu, kor);
    if (lane == 0) {
        warp_red[0][warp_id] = kand;
        warp_red[1][warp_id] = kor;
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t a = 0xffffffffu, o = 0u;
        for (int w = 0; w < kTopkWarps; ++w) {
            a &= warp_red[0][w];
            o |= warp_red[1][w];
        }
        const int lead = __clz(a ^ o);  // bits every key shares (32: all keys equal)
        warp_red[0][0] = (uint32_t)lead;
        s_prefix = lead >= 32 ? a : (a & ~(0xffffffffu >> lead));
        s_kleft = (uint32_t)k;
    }
    __syncthreads();
    const int lead = (int)warp_red[0][0];
    TOPK_TRACE(1);
    auto key_at = [&](int64_t j) -> uint32_t { return stage_row ? keys[j] : ord_key(src[j]); };

    // radix select over the differing bits only, 8 bits per pass from the top
    __shared__ uint32_t whist[kTopkWarps][256];
    uint32_t mask = lead >= 32 ? 0xffffffffu : ~(0xffffffffu >> lead);
    int pass = 0;
    for (int top = 32 - lead; top > 0; top -= 8, ++pass) {
        const int nb = min(8, top), shift = top - nb;
        const uint32_t dmask = (1u << nb) - 1u;
        for (int i = tid; i < kTopkWarps * 256; i += kTopkThreads) (&whist[0][0])[i] = 0;
        __syncthreads();
        const uint32_t prefix = s_prefix;
        uint32_t* wh = whist[warp_id];
        for (int64_t j = tid; j < m; j += kTopkThreads) {
            const uint32_t o = key_at(j);
            if ((o & mask) == prefix) atomicAdd(&wh[(o >> shift) & dmask], 1u);
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
        mask |= dmask << shift;
        __syncthreads();
        TOPK_TRACE(2 + min(pass, 3));
    }
    const uint32_t T = s_prefix;
    const uint32_t need_eq = s_kleft;           // ties to take, lowest index first
    const uint32_t G = (uint32_t)k - need_eq;   // strictly greater

    // collect, in index order: warp w owns the contiguous segment [w*seg, (w+1)*seg); one
    // counting pass (ballots), one block scan of the per-warp counts, one write pass
    const int64_t seg = ((m + kTopkWarps * 32 - 1) / (kTopkWarps * 32)) * 32;
    const int64_t s0 = warp_id * seg, s1 = min(m, s0 + seg);
    uint32_t n_gt = 0, n_eq = 0;
    for (int64_t j0 = s0; j0 < s1; j0 += 32) {
        const int64_t j = j0 + lane;
        const uint32_t o = j < s1 ? key_at(j) : 0u;
        n_gt += __popc(__ballot_sync(0xffffffffu, j < s1 && o > T));
        n_eq += __popc(__ballot_sync(0xffffffffu, j < s1 && o == T));
    }
    if (lane == 0) {
        warp_tot[0][warp_id] = n_gt;
        warp_tot[1][warp_id] = n_eq;
    }
    __syncthreads();
    if (tid < 32) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const uint32_t v = tid < kTopkWarps ? warp_tot[q][tid] : 0u;
            uint32_t incl = v;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += t;
            }
            __syncwarp();
            if (tid < kTopkWarps) warp_tot[q][tid] = incl - v;  // exclusive offsets
        }
    }
    __syncthreads();
    uint32_t gt_run = warp_tot[0][warp_id], eq_run = warp_tot[1][warp_id];
    for (int64_t j0 = s0; j0 < s1; j0 += 32) {
        const int64_t j = j0 + lane;
        const uint32_t o = j < s1 ? key_at(j) : 0u;
        const bool gt = j < s1 && o > T, eq = j < s1 && o == T;
        const uint64_t comp = ((uint64_t)o << 32) | (uint32_t)~(uint32_t)j;
        const uint32_t lt_mask = (1u << lane) - 1u;
        const uint32_t gb = __ballot_sync(0xffffffffu, gt);
        if (gt) sel[gt_run + __popc(gb & lt_mask)] = comp;
        gt_run += __popc(gb);
        const uint32_t eb = __ballot_sync(0xffffffffu, eq);
        const uint32_t r = eq_run + __popc(eb & lt_mask);
        if (eq && r < need_eq) sel[G + r] = comp;
        eq_run += __popc(eb);
    }
    __syncthreads();
    TOPK_TRACE(6);
    int32_t* dst = idx_out + row * k;
    if (!sorted) {  // the exact set: strictly-greater then ties, each in index order
        for (int i = tid; i < k; i += kTopkThreads) dst[i] = (int32_t)(~(uint32_t)sel[i]);
        if (tid == 0 && counts) counts[row] = (int32_t)k;
        return;
    }
    if (k <= 256) {
        // small k: all composites are distinct, output slot = number of selected composites
        // above it (O(k^2 / threads) compares)
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
    bitonic_sort_desc(sel, sort_pow2);
    TOPK_TRACE(7);
    for (int i = tid; i < k; i += kTopkThreads) dst[i] = (int32_t)(~(uint32_t)sel[i]);
    if (tid == 0 && counts) counts[row] = (int32_t)k;
}

// ---------------------------------------------------------------------------
// Cluster top-k for few, long rows (the MLP selection: 24 rows x 12288 at FLUX would keep
// only 24 SMs busy): a cluster of CS CTAs shares one row.  Each CTA owns a contiguous
// segment (its warps contiguous sub-segments, so index order = (CTA, warp, lane) order);
// every radix pass builds per-warp histograms, sums them per CTA, and every CTA reads all
// CTAs' histograms through distributed shared memory to take the same digit decision.  The
// per-CTA / per-warp counts above the selected digit accumulate into exact gt / eq offsets,
// so one write pass emits the index SET (strictly greater, then the lowest-index ties), each
// part in index order.  Unsorted output only (the PROD block path).
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(cta));
    return r;
}
// Remote shared-memory stores that complete_tx on the receiver's mbarrier: the histogram
// exchange needs no cluster-wide barrier (barrier.cluster.arrive.release compiles to
// MEMBAR.ALL.GPU + CCTL.IVALL per pass)
__device__ __forceinline__ void st_async_v4(uint32_t raddr, uint4 v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
                 ::"r"(raddr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar) : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t raddr, uint32_t a, uint32_t b, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];"
                 ::"r"(raddr), "r"(a), "r"(b), "r"(rbar) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// Fused MLP selection scores (mlp.cpp:116): score = |sum_s partial[s] - cached| in the same
// fixed summation order as k_means_reduce, so the keys are bit-identical to the unfused path.
struct TopkFusedScores {
    const float* partial;  // [ks][rows * m]
    int ks;
    const float* cached;   // [rows * m]
};

template <int CS, bool kFused>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(kTopkThreads)
k_topk_cluster(const float* __restrict__ scores, int64_t m, int64_t k, int32_t* __restrict__ idx_out,
               int32_t* __restrict__ counts, TopkFusedScores fs) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint32_t* keys = reinterpret_cast<uint32_t*>(smem);  // this CTA's segment
    __shared__ uint32_t whist[kTopkWarps][256];
    // every CTA's histogram, double-buffered by pass: slot [rank] written locally, the peers'
    // slots by their st.async pushes (mb[pass & 1]); AND / OR of the keys likewise (mb[2])
    __shared__ __align__(16) uint32_t rhist[2][CS][256];
    __shared__ __align__(8) uint32_t rred[CS][2];
    __shared__ __align__(8) uint64_t mb[3];
    __shared__ uint32_t s_prefix, s_kleft, s_sel, s_shift;
    __shared__ uint32_t cta_gt[CS], warp_gt[kTopkWarps], warp_eq[kTopkWarps], cta_eq[CS];
    __shared__ uint32_t tot_bins[256];
    pdl_wait();
    if (threadIdx.x == 0) pdl_trigger();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t rank = cluster_rank();
    if (tid == 0) {
        for (int i = 0; i < 3; ++i) tc::mbar_init(&mb[i], 1);
        tc::fence_barrier_init();
    }
    cluster_arrive_relaxed();  // waited for after the load phase: the peers' barriers exist
    const int64_t row = blockIdx.x / CS;
    const float* src = scores + row * m;
    TOPK_TRACE(0);
    const int64_t seg = (m + CS - 1) / CS;
    const int64_t c0 = (int64_t)rank * seg, c1 = min(m, c0 + seg);
    const int64_t nloc = max((int64_t)0, c1 - c0);
    const int64_t wseg = (nloc + kTopkWarps - 1) / kTopkWarps;  // per-warp sub-segment
    const int64_t w0 = min(nloc, warp * wseg), w1 = min(nloc, w0 + wseg);
    uint32_t kand = 0xffffffffu, kor = 0u;
    // kU elements per lane per round, every load of the round issued before the first use
    // (the scores are an L2-latency-bound read: one round covers FLUX's 192 per warp)
    constexpr int kU = 8;
    for (int64_t jb = w0 + lane; jb < w1; jb += 32 * kU) {
        float sc[kU];
        if constexpr (kFused) {
            const int64_t total = (int64_t)gridDim.x / CS * m, e0 = row * m + c0 + jb;
            float cv[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const bool ok = jb + u * 32 < w1;
                sc[u] = ok ? __ldg(fs.partial + e0 + u * 32) : 0.f;
                cv[u] = ok ? __ldg(fs.cached + e0 + u * 32) : 0.f;
            }
            for (int q = 1; q < fs.ks; ++q) {
                const float* pq = fs.partial + (int64_t)q * total + e0;
#pragma unroll
                for (int u = 0; u < kU; ++u)
                    if (jb + u * 32 < w1) sc[u] += __ldg(pq + u * 32);
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) sc[u] = fabsf(sc[u] - cv[u]);
        } else {
#pragma unroll
            for (int u = 0; u < kU; ++u) sc[u] = jb + u * 32 < w1 ? __ldg(src + c0 + jb + u * 32) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if (jb + u * 32 < w1) {
                const uint32_t o = ord_key(sc[u]);
                keys[jb + u * 32] = o;
                kand &= o;
                kor |= o;
            }
        }
    }
    kand = __reduce_and_sync(0xffffffffu, kand);
    kor = __reduce_or_sync(0xffffffffu, kor);
    if (lane == 0) { whist[0][warp] = kand; whist[1][warp] = kor; }
    if (tid < CS) { cta_gt[tid] = 0; cta_eq[tid] = 0; }
    if (tid < kTopkWarps) warp_gt[tid] = 0;
    __syncthreads();
    cluster_wait();
    if (tid == 0) {
        uint32_t a = 0xffffffffu, o = 0u;
        for (int w = 0; w < kTopkWarps; ++w) { a &= whist[0][w]; o |= whist[1][w]; }
        rred[rank][0] = a;
        rred[rank][1] = o;
        tc::mbar_arrive_expect_tx(&mb[2], (CS - 1) * 8);
        for (uint32_t r = 1; r < CS; ++r) {
            const uint32_t pr = (rank + r) % CS;
            st_async_v2(mapa_u32(smem_u32_generic(&rred[rank][0]), pr), a, o, mapa_u32(smem_u32_generic(&mb[2]), pr));
        }
        tc::mbar_wait(&mb[2], 0);
        for (uint32_t r = 0; r < CS; ++r) { a &= rred[r][0]; o |= rred[r][1]; }
        const int lead = __clz(a ^ o);
        s_prefix = lead >= 32 ? a : (a & ~(0xffffffffu >> lead));
        s_kleft = (uint32_t)k;
        s_shift = (uint32_t)lead;
    }
    __syncthreads();
    const int lead = (int)s_shift;
    TOPK_TRACE(1);
    uint32_t mask = lead >= 32 ? 0xffffffffu : ~(0xffffffffu >> lead);
    int pass = 0;
    for (int top = 32 - lead; top > 0; top -= 8, ++pass) {
        const int nb = min(8, top), shift = top - nb;
        const uint32_t dmask = (1u << nb) - 1u;
        const int hb = pass & 1;
        TOPK_TRACE(2 + min(pass, 3));
        for (int i = tid; i < kTopkWarps * 256; i += kTopkThreads) (&whist[0][0])[i] = 0;
        __syncthreads();
        const uint32_t prefix = s_prefix;
        for (int64_t j = w0 + lane; j < w1; j += 32) {
            const uint32_t o = keys[j];
            if ((o & mask) == prefix) atomicAdd(&whist[warp][(o >> shift) & dmask], 1u);
        }
        __syncthreads();
        for (int i = tid; i < 256; i += kTopkThreads) {
            uint32_t acc = 0;
#pragma unroll
            for (int w = 0; w < kTopkWarps; ++w) acc += whist[w][i];
            rhist[hb][rank][i] = acc;
        }
        __syncthreads();
        // push this CTA's histogram to the peers (64 x 16 B each); a peer is at most one pass
        // ahead (it needs this CTA's push of the pass it is on), so two buffers suffice
        if (tid == 0) tc::mbar_arrive_expect_tx(&mb[hb], (CS - 1) * 1024);
        if (tid < 64 * (CS - 1)) {
            const uint32_t pr = (rank + 1 + tid / 64) % CS;
            const int q = tid % 64;
            const uint4 v = *reinterpret_cast<const uint4*>(&rhist[hb][rank][q * 4]);
            st_async_v4(mapa_u32(smem_u32_generic(&rhist[hb][rank][q * 4]), pr), v,
                        mapa_u32(smem_u32_generic(&mb[hb]), pr));
        }
        tc::mbar_wait(&mb[hb], (pass >> 1) & 1);
        // thread = bin: its per-CTA counts and the total
        uint32_t vr[CS];
        uint32_t vtot = 0;
        if (tid < 256) {
#pragma unroll
            for (int r = 0; r < CS; ++r) {
                vr[r] = rhist[hb][r][tid];
                vtot += vr[r];
            }
            tot_bins[tid] = vtot;
        }
        __syncthreads();
        if (tid < 32) {
            // lane l owns descending digits d = 8l..8l+7 (bin = 255 - d), summed over the cluster
            uint32_t cnt[8], tot = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                cnt[i] = tot_bins[255 - (8 * tid + i)];
                tot += cnt[i];
            }
            uint32_t incl = tot;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += t;
            }
            uint32_t run = incl - tot;
            const uint32_t need = s_kleft;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (run < need && run + cnt[i] >= need) {
                    s_sel = (uint32_t)(255 - (8 * tid + i));
                    s_kleft = need - run;
                }
                run += cnt[i];
            }
        }
        __syncthreads();
        const uint32_t sel = s_sel;
        // counts of this pass's digits above the selected one (strictly greater than the final
        // threshold), per CTA and per warp of this CTA; the selected bin's counts are the ties
        // once the last pass has run
        if (tid < 256) {  // warps 0..7 cover the 256 bins: per-CTA sums by warp reduction
            const bool above = (uint32_t)tid > sel && (uint32_t)tid <= dmask;
#pragma unroll
            for (int r = 0; r < CS; ++r) {
                const uint32_t g = __reduce_add_sync(0xffffffffu, above ? vr[r] : 0u);
                if (lane == 0 && g) atomicAdd(&cta_gt[r], g);
            }
        }
        {   // each warp sums its own histogram's bins above the selected digit
            uint32_t g = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t d = (uint32_t)(lane * 8 + i);
                if (d > sel && d <= dmask) g += whist[warp][d];
            }
            g = __reduce_add_sync(0xffffffffu, g);
            if (lane == 0) warp_gt[warp] += g;
        }
        if ((uint32_t)tid == sel) {
#pragma unroll
            for (int r = 0; r < CS; ++r) cta_eq[r] = vr[r];
        }
        if (tid < kTopkWarps) warp_eq[tid] = whist[tid][sel];
        if (tid == 0) s_prefix = prefix | (sel << shift);
        mask |= dmask << shift;
        __syncthreads();
    }
    if (lead >= 32) {  // every key equal: all ties
        if (tid < CS) { cta_gt[tid] = 0; cta_eq[tid] = (uint32_t)max((int64_t)0, min(m, (int64_t)(tid + 1) * seg) - (int64_t)tid * seg); }
        if (tid < kTopkWarps) { warp_gt[tid] = 0; warp_eq[tid] = (uint32_t)(min(nloc, (tid + 1) * wseg) - min(nloc, tid * wseg)); }
        __syncthreads();
    }
    TOPK_TRACE(6);
    const uint32_t T = s_prefix;
    const uint32_t need_eq = s_kleft;
    const uint32_t G = (uint32_t)k - need_eq;
    // offsets: CTAs before this one, then warps before this one (index order)
    uint32_t gt_off = 0, eq_off = 0;
    for (uint32_t r = 0; r < rank; ++r) { gt_off += cta_gt[r]; eq_off += cta_eq[r]; }
    for (int w = 0; w < warp; ++w) { gt_off += warp_gt[w]; eq_off += warp_eq[w]; }
    int32_t* dst = idx_out + row * k;
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (int64_t j0 = w0; j0 < w1; j0 += 32) {
        const int64_t j = j0 + lane;
        const uint32_t o = j < w1 ? keys[j] : 0u;
        const bool gt = j < w1 && o > T, eq = j < w1 && o == T;
        const uint32_t gb = __ballot_sync(0xffffffffu, gt);
        if (gt) dst[gt_off + __popc(gb & lt_mask)] = (int32_t)(c0 + j);
        gt_off += __popc(gb);
        const uint32_t eb = __ballot_sync(0xffffffffu, eq);
        const uint32_t r = eq_off + __popc(eb & lt_mask);
        if (eq && r < need_eq) dst[G + r] = (int32_t)(c0 + j);
        eq_off += __popc(eb);
    }
    if (rank == 0 && tid == 0 && counts) counts[row] = (int32_t)k;
    TOPK_TRACE(7);
    // no trailing cluster barrier: peers never read this CTA's shared memory, and every
    // push this CTA receives has been waited for
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

bool topk_cluster_eligible(int64_t rows, int64_t m) {
    return rows * 4 <= 148 && m >= 4 * kTopkThreads && (m + 3) / 4 * 4 <= 48 * 1024;
}

// Unsorted top-k of |sum_s partial[s] - cached| (the MLP change scores) without materialising
// the scores: the split-K reduction of the tile means runs inside the top-k load.
cudaError_t topk_rows_fused_absdiff(const float* partial, int ks, const float* cached, int64_t rows,
                                    int64_t m, int64_t k, int32_t* idx, int32_t* counts,
                                    cudaStream_t s) {
    if (!topk_cluster_eligible(rows, m)) return cudaErrorNotSupported;
    const size_t csm = sizeof(uint32_t) * (size_t)((m + 3) / 4);
    {
        cudaError_t e = ensure_smem_attr(k_topk_cluster<4, true>, 196 * 1024);
        if (e != cudaSuccess) return e;
    }
    return launch_ex(k_topk_cluster<4, true>, dim3((unsigned)(rows * 4)), dim3(kTopkThreads), csm, s, 1,
                     (const float*)nullptr, m, k, idx, counts, TopkFusedScores{partial, ks, cached});
}

cudaError_t topk_rows(const float* scores, int64_t rows, int64_t m, int64_t k, int32_t* idx,
                      int32_t* counts, cudaStream_t s, bool sorted) {
    if (rows == 0) return cudaSuccess;
    if (k > kTopkMaxSortK) return cudaErrorNotSupported;  // caller uses topk_rows_global
    if (!sorted && topk_cluster_eligible(rows, m)) {
        // few long rows: a cluster of 4 CTAs per row (unsorted index set)
        const size_t csm = sizeof(uint32_t) * (size_t)((m + 3) / 4);
        {
            cudaError_t e = ensure_smem_attr(k_topk_cluster<4, false>, 196 * 1024);
            if (e != cudaSuccess) return e;
        }
        return launch_ex(k_topk_cluster<4, false>, dim3((unsigned)(rows * 4)), dim3(kTopkThreads), csm, s,
                         1, scores, m, k, idx, counts, TopkFusedScores{});
    }
    int p2 = 64;  // the register runs of the bitonic sort work on 64-element segments
    while (p2 < k) p2 <<= 1;
    const int stage = m <= kTopkMaxSmemRow ? 1 : 0;
    const size_t smem = sizeof(uint64_t) * p2 + (stage ? sizeof(float) * m : 0);
    {
        cudaError_t e = ensure_smem_attr(k_topk_rows, 196 * 1024);
        if (e != cudaSuccess) return e;
    }
    return launch_ex(k_topk_rows, dim3((unsigned)rows), dim3(kTopkThreads), smem, s, 1, scores, m, k, idx,
                     counts, stage, p2, sorted ? 1 : 0);
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
    {
        cudaError_t e = ensure_smem_attr(k_validate, 200 * 1024);
        if (e != cudaSuccess) return e;
    }
    k_validate<<<(unsigned)rows, 256, smem, s>>>(idx, counts, k_max, domain, flags);
    return cudaGetLastError();
}

}  // namespace dev
}  // namespace csd

// Debug only: phase timeline of CTA 0 of the next top-k launches (8 uint64 slots).
extern "C" int csd_debug_set_topk_trace(void* dev_buf) {
    uint64_t* p = static_cast<uint64_t*>(dev_buf);
    return cudaMemcpyToSymbol(csd::dev::g_topk_trace, &p, sizeof(p)) == cudaSuccess ? 0 : 7;
}
