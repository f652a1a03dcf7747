// attn_px.cu — column-sparse delta attention with P staged in SHARED memory (CSD_MODE_PROD).
//
// Replaces sparse_delta_attention (attention.cpp:147-194) for query chunks of 129..192 rows,
// E = 128 (FLUX / Hunyuan chunk 192), out = base + scale * softmax(Q_c K_S^T / sqrt(E)) V_S.
//
// Same work split as k_attn_pp (attn_pp.cu): item = (b, h, chunk) as two M-tiles of 128 rows
// sharing every gathered K/V block; one softmax warpgroup per tile, one thread per query row
// holding the block's 128 key columns.  The difference is where P lives.  In k_attn_pp P is
// written over S in TMEM (TS-form P V), so S_t(j+1) can only be issued once P_t V_j has
// consumed P_t(j): every key block pays softmax + P V + S in series (measured: 2.6k + 1.8k
// cycles per block).  Here the softmax warps store P_t(j) into a shared-memory
// A operand (SS-form P V), so the S_t buffer is free as soon as the softmax has LOADED S_t(j)
// into registers: S_t(j+1) is issued then (barrier bar_sl) and lands while the exponentials
// of block j run -- the next softmax starts right after this one.  P_t's single smem buffer
// is rewritten only after P_t V_{j-1} completed (bar_pv), which the exponentials cover.
//
// TMEM (512 columns): S_0 [0,128), S_1 [128,256), O_0 [256,384), O_1 [384,512).
// SMEM: Q_0 32 KB, Q_1 16 KB (64 rows; the MMA's dead rows 64-127 read the next region),
// P_0 32 KB, P_1 16 KB (same), K ring 2 x 32 KB, V ring 2 x 32 KB.  The epilogue combines
// out = base + scale O / l straight from global memory (the base tile is prefetched into L2
// when the item's Q is loaded).
//
// Roles (16 warps): warp 0 lane 0 Q loader + base L2 prefetch; warp 1 MMA issuer; warps 2,
// 12-15 K/V row gathers (cp.async); warps 4-7 softmax tile 0, warps 8-11 softmax tile 1.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "launch_util.h"
#include "tc_common.cuh"

namespace csd {
namespace dev {

using namespace csd::tc;

bool make_map_bf16(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows,
                   uint64_t pitch_elems, uint32_t box_rows);

namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale O only when the max grows > 2^8
constexpr int E = 128;
constexpr uint32_t kThreads = 512;
constexpr int kCopyThreads = 160;  // warps 2, 12-15
constexpr uint32_t kStrip = 128 * 128;  // 128 rows x 128 B
constexpr uint32_t kKV = 2 * kStrip;    // one K or V block (2 strips)
constexpr uint32_t kOffQ0 = 0, kOffQ1 = 32768, kOffP0 = 49152, kOffP1 = 81920;
constexpr uint32_t kOffK = 98304, kOffV = kOffK + 2 * kKV, kOffBar = kOffV + 2 * kKV;
constexpr uint32_t kSmemBytes = kOffBar + 256;  // 229,632 B (<= 227 KB)

struct PXParams {
    const int32_t* idx;
    const int32_t* counts;
    int64_t k_max;
    const __nv_bfloat16* kp;
    const __nv_bfloat16* vp;
    const __nv_bfloat16* base;
    __nv_bfloat16* out;
    float scale;
    float qk_scale_log2;
    int layout;
    int heads, n, chunk, chunks, items;
    int rows1;  // live rows of M-tile 1 (chunk - 128)
};

__device__ __forceinline__ int64_t px_tok_off(int layout, int64_t b, int64_t h, int64_t tok, int heads, int n) {
    return layout == CSD_LAYOUT_BHNE ? (((b * heads + h) * (int64_t)n) + tok) * E
                                     : ((b * (int64_t)n + tok) * heads + h) * E;
}

__global__ void __launch_bounds__(kThreads, 1)
k_attn_px(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_b, const PXParams p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_u32 = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int items = p.items;
    const int rows_t[2] = {128, p.rows1};
    const int lw0 = 4, lw1 = (p.rows1 + 31) >> 5;  // live softmax warps per tile

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
    uint64_t* bar_q = bars + 0;    // [2] Q_t landed
    uint64_t* bar_qe = bars + 2;   // [2] Q_t free (the item's last S_t completed)
    uint64_t* bar_kf = bars + 4;   // [2] K ring slot full (cp.async)
    uint64_t* bar_ke = bars + 6;   // [2] K ring slot free
    uint64_t* bar_vf = bars + 8;   // [2]
    uint64_t* bar_ve = bars + 10;  // [2]
    uint64_t* bar_s = bars + 12;   // [2] S_t in TMEM
    uint64_t* bar_sl = bars + 14;  // [2] S_t loaded into the softmax registers (buffer free)
    uint64_t* bar_p = bars + 16;   // [2] P_t in shared memory (and O_t rescaled)
    uint64_t* bar_pv = bars + 18;  // [2] P_t V of the block completed (P_t buffer free)
    uint64_t* bar_o = bars + 20;   // [2] O_t final for the item
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22);
    uint8_t* const sk = smem + kOffK;
    uint8_t* const sv = smem + kOffV;
    if (threadIdx.x == 0) {
        if ((raw_u32 & 1023u) != 0) __trap();  // the host sizes the request without slack
        for (int i = 0; i < 2; ++i) {
            const uint32_t lw = i == 0 ? lw0 : lw1;
            mbar_init(bar_q + i, 1);
            mbar_init(bar_qe + i, 1);
            mbar_init(bar_kf + i, kCopyThreads);
            mbar_init(bar_ke + i, 1);
            mbar_init(bar_vf + i, kCopyThreads);
            mbar_init(bar_ve + i, 1);
            mbar_init(bar_s + i, 1);
            mbar_init(bar_sl + i, 32u * lw);
            mbar_init(bar_p + i, 32u * lw);
            mbar_init(bar_pv + i, 1);
            mbar_init(bar_o + i, 1);
        }
        fence_barrier_init();
    }
    auto count_of = [=](int pos) -> int { return p.counts[pos]; };
    auto next_live = [=](int from, int& cnt_out) -> int {
        int x = from;
        cnt_out = 0;
        for (; x < items; x += gridDim.x) {
            cnt_out = count_of(x);
            if (cnt_out > 0) break;
        }
        return x;
    };
    auto item_rows = [=](int it, int& row_base, int& col0) {
        const int bh = it / p.chunks;
        row_base = p.layout == CSD_LAYOUT_BHNE ? bh * p.n : (bh / p.heads) * p.n;
        col0 = p.layout == CSD_LAYOUT_BHNE ? 0 : (bh % p.heads) * E;
        row_base += (it % p.chunks) * p.chunk;
    };
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    if (threadIdx.x == 0) pdl_trigger();

    if (warp < 4 || warp >= 12) {
        regs_dec<72>();
        if (warp == 0) {
            if (lane == 0) {
                // ---------------------------------------------------- Q loader
                tma_prefetch_desc(&tm_q);
                const int qrows[2] = {128, (p.rows1 + 63) / 64 * 64};
                const uint32_t offq[2] = {kOffQ0, kOffQ1}, qstrip[2] = {kStrip, (uint32_t)qrows[1] * 128u};
                uint32_t li = 0;
                int cnt = 0;
                for (int it = next_live(blockIdx.x, cnt); it < items; ++li) {
                    int r0, col0;
                    item_rows(it, r0, col0);
                    for (int t = 0; t < 2; ++t) {
                        if (li > 0) mbar_wait(bar_qe + t, (li - 1) & 1);
                        mbar_arrive_expect_tx(bar_q + t, 2u * (uint32_t)qrows[t] * 128u);
                        for (int hf = 0; hf < 2; ++hf)
                            for (int bx = 0; bx < qrows[t] / 64; ++bx)
                                tma_load_2d(&tm_q, bar_q + t, smem + offq[t] + hf * qstrip[t] + bx * 8192,
                                            col0 + hf * 64, r0 + t * 128 + bx * 64);
                    }
                    // this item's base rows into L2 for the epilogue; the next item's Q too
                    for (int hf = 0; hf < 2; ++hf)
                        for (int bx = 0; bx < (p.chunk + 63) / 64; ++bx)
                            tma_prefetch_2d(&tm_b, col0 + hf * 64, r0 + bx * 64);
                    const int nx = next_live(it + gridDim.x, cnt);
                    if (nx < items) {
                        int nr0, ncol0;
                        item_rows(nx, nr0, ncol0);
                        for (int hf = 0; hf < 2; ++hf)
                            for (int bx = 0; bx < (p.chunk + 63) / 64; ++bx)
                                tma_prefetch_2d(&tm_q, ncol0 + hf * 64, nr0 + bx * 64);
                    }
                    it = nx;
                }
            }
        } else if (warp == 1) {
            // -------------------------------------------------------- MMA issuer
            constexpr uint32_t idS = idesc_bf16(128, 128, false, false);
            constexpr uint32_t idO = idesc_bf16(128, E, false, true);
            const uint32_t sQ = smem_u32(smem), sK = smem_u32(sk), sV = smem_u32(sv);
            const uint32_t offq[2] = {kOffQ0, kOffQ1}, qstrip[2] = {kStrip, (uint32_t)((p.rows1 + 63) / 64 * 64) * 128u};
            const uint32_t offp[2] = {kOffP0, kOffP1}, pstrip[2] = {qstrip[0], qstrip[1]};
            struct Cur {
                int it, cnt, nblk, j;
                uint32_t li, g;
            };
            auto start = [&](Cur& c) {
                c.it = next_live(blockIdx.x, c.cnt);
                c.nblk = (c.cnt + 127) >> 7;
                c.j = 0;
                c.li = 0;
                c.g = 0;
            };
            auto advance = [&](Cur& c) {
                ++c.g;
                if (++c.j == c.nblk) {
                    c.it = next_live(c.it + gridDim.x, c.cnt);
                    c.nblk = (c.cnt + 127) >> 7;
                    c.j = 0;
                    ++c.li;
                }
            };
            auto commit = [&](uint64_t* b) {
                if (elect_one()) mma_commit(b);
                __syncwarp();
            };
            auto issue_s = [&](int t, const Cur& c) {  // S_t(c.g) = Q_t K(c.g)^T
                if (c.j == 0) mbar_wait(bar_q + t, c.li & 1);
                mbar_wait(bar_kf + (c.g & 1), (c.g >> 1) & 1);
                fence_proxy_async_smem();  // cp.async (generic proxy) -> tcgen05 reads
                tc_fence_after();
                const uint32_t qb = sQ + offq[t], kb = sK + (c.g & 1) * kKV;
                uint64_t da[E / 16], db[E / 16];
#pragma unroll
                for (int kk = 0; kk < E / 16; ++kk) {
                    da[kk] = desc_kmajor_sw128(qb + (kk / 4) * qstrip[t] + (kk % 4) * 32);
                    db[kk] = desc_kmajor_sw128(kb + (kk / 4) * kStrip + (kk % 4) * 32);
                }
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < E / 16; ++kk)
                        mma_bf16(tmem + t * 128, da[kk], db[kk], idS, kk > 0 ? 1u : 0u);
                    mma_commit(bar_s + t);
                    if (c.j == c.nblk - 1) mma_commit(bar_qe + t);
                    if (t == 1) mma_commit(bar_ke + (c.g & 1));  // both tiles' S read the K slot
                }
                __syncwarp();
            };
            Cur cs, cv;
            start(cs);
            start(cv);
            if (cs.it < items) {
                issue_s(0, cs);
                issue_s(1, cs);
                advance(cs);
            }
            while (cv.it < items) {
                const uint32_t g = cv.g;
                // the next block's S as soon as each tile's softmax holds S(g) in registers
                if (cs.it < items) {
                    mbar_wait(bar_sl + 0, g & 1);
                    issue_s(0, cs);
                    mbar_wait(bar_sl + 1, g & 1);
                    issue_s(1, cs);
                    advance(cs);
                }
                // P_t V(g) once P_t is in shared memory
                mbar_wait(bar_vf + (g & 1), (g >> 1) & 1);
                for (int t = 0; t < 2; ++t) {
                    mbar_wait(bar_p + t, g & 1);
                    fence_proxy_async_smem();  // softmax st.shared of P -> tcgen05 reads
                    tc_fence_after();
                    const uint32_t pb = sQ + offp[t], vb = sV + (g & 1) * kKV;
                    uint64_t dp[8], dv[8];
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        dp[kk] = desc_kmajor_sw128(pb + (kk / 4) * pstrip[t] + (kk % 4) * 32);
                        dv[kk] = desc_mnmajor_sw128(vb + kk * 2048, kStrip);
                    }
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)
                            mma_bf16(tmem + 256 + t * 128, dp[kk], dv[kk], idO, (cv.j > 0 || kk > 0) ? 1u : 0u);
                        mma_commit(bar_pv + t);
                        if (t == 1) mma_commit(bar_ve + (g & 1));
                        if (cv.j == cv.nblk - 1) mma_commit(bar_o + t);
                    }
                    __syncwarp();
                }
                advance(cv);
            }
            (void)commit;
        } else if (warp == 2 || warp >= 12) {
            // -------------------------------------------------------- sparse K/V row copies
            constexpr int kRowStep = kCopyThreads / (E / 8);
            constexpr int kCpRows = (128 + kRowStep - 1) / kRowStep;
            const int ct = warp == 2 ? lane : 32 + (warp - 12) * 32 + lane;
            const int c16 = ct % (E / 8), r0 = ct / (E / 8);
            const uint32_t cbase = (uint32_t)(c16 >> 3) * kStrip;
            const int64_t rs = p.layout == CSD_LAYOUT_BHNE ? E : (int64_t)p.heads * E;
            const uint32_t sKs = smem_u32(sk), sVs = smem_u32(sv);
            auto load_ids = [=](int it, int cnt, int j, int32_t (&id)[kCpRows]) {
                const int32_t* ids = p.idx + (int64_t)(it < items ? it : 0) * p.k_max;
#pragma unroll
                for (int i = 0; i < kCpRows; ++i) {
                    const int r = j * 128 + r0 + kRowStep * i;
                    id[i] = (it < items && r0 + kRowStep * i < 128 && r < cnt) ? __ldg(ids + r) : -1;
                }
            };
            int cnt = 0;
            int it = next_live(blockIdx.x, cnt), j = 0;
            int nx_cnt = 0;
            int nx_it = it < items ? next_live(it + gridDim.x, nx_cnt) : items;
            int32_t id[kCpRows];
            load_ids(it, cnt, 0, id);
            for (uint32_t g = 0; it < items; ++g) {
                const int bh = it / p.chunks;
                const int64_t o0 = px_tok_off(p.layout, bh / p.heads, bh % p.heads, 0, p.heads, p.n) + c16 * 8;
                const __nv_bfloat16* kb = p.kp + o0;
                const __nv_bfloat16* vb = p.vp + o0;
                const int nblk = (cnt + 127) / 128;
                int nit = it, ncnt = cnt, nj = j + 1;
                if (nj == nblk) {
                    nit = nx_it;
                    ncnt = nx_cnt;
                    nj = 0;
                }
                const int s = g & 1;
                if (g >= 2) mbar_wait(bar_ke + s, ((g >> 1) - 1) & 1);
#pragma unroll
                for (int i = 0; i < kCpRows; ++i) {
                    const uint32_t row = (uint32_t)(r0 + kRowStep * i);
                    if (row < 128u)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                                         sKs + s * kKV + cbase + sw128_offset(row, (uint32_t)(c16 & 7))),
                                     "l"(kb + (id[i] >= 0 ? (int64_t)id[i] * rs : 0)), "r"(id[i] >= 0 ? 16u : 0u)
                                     : "memory");
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar_kf + s))
                             : "memory");
                int32_t idn[kCpRows];
                load_ids(nit, ncnt, nj, idn);
                if (nj == 0 && nit < items) nx_it = next_live(nit + gridDim.x, nx_cnt);
                if (g >= 2) mbar_wait(bar_ve + s, ((g >> 1) - 1) & 1);
#pragma unroll
                for (int i = 0; i < kCpRows; ++i) {
                    const uint32_t row = (uint32_t)(r0 + kRowStep * i);
                    if (row < 128u)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                                         sVs + s * kKV + cbase + sw128_offset(row, (uint32_t)(c16 & 7))),
                                     "l"(vb + (id[i] >= 0 ? (int64_t)id[i] * rs : 0)), "r"(id[i] >= 0 ? 16u : 0u)
                                     : "memory");
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar_vf + s))
                             : "memory");
#pragma unroll
                for (int i = 0; i < kCpRows; ++i) id[i] = idn[i];
                it = nit;
                cnt = ncnt;
                j = nj;
            }
        }
    } else {
        regs_inc<184>();
        // ------------------------------------------------------------ softmax + epilogue
        const int t = (warp - 4) >> 2, quad = (warp - 4) & 3;
        const int row = quad * 32 + lane;  // TMEM lane = row of tile t
        const int crow = t * 128 + row;    // row within the item
        const bool row_ok = row < rows_t[t];
        if (quad * 32 < rows_t[t]) {
            const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
            const uint32_t tS = tmem + lane_off + t * 128;
            const uint32_t tO = tmem + lane_off + 256 + t * 128;
            // P_t: K-major 128B-swizzled A operand, strip = 64 keys; this thread's row
            uint8_t* const prow = smem + (t == 0 ? kOffP0 : kOffP1) + row * 128;
            const uint32_t pstrip = t == 0 ? kStrip : (uint32_t)((p.rows1 + 63) / 64 * 64) * 128u;
            const float sl2 = p.qk_scale_log2;
            const bool has_base = p.base != nullptr;
            uint32_t g = 0, li = 0;
            int cnt_nx = blockIdx.x < items ? count_of(blockIdx.x) : 0;
            for (int it = blockIdx.x; it < items; it += gridDim.x) {
                const int cnt = cnt_nx;
                if (it + (int)gridDim.x < items) cnt_nx = count_of(it + gridDim.x);
                const int c = it % p.chunks, bh = it / p.chunks;
                const int b = bh / p.heads, h = bh % p.heads;
                const int64_t tok = (int64_t)c * p.chunk + crow;
                const int64_t off = px_tok_off(p.layout, b, h, tok, p.heads, p.n);
                if (cnt == 0) {  // pass base through (attention.cpp:169)
                    if (row_ok && has_base && p.base != p.out) {
                        const uint4* src = reinterpret_cast<const uint4*>(p.base + off);
                        uint4* dst = reinterpret_cast<uint4*>(p.out + off);
#pragma unroll
                        for (int q = 0; q < E / 8; ++q) dst[q] = src[q];
                    }
                    continue;
                }
                const int nblk = (cnt + 127) / 128;
                float m_run = -INFINITY, l_run = 0.f;
                for (int j = 0; j < nblk; ++j, ++g) {
                    const int ncols = min(128, cnt - j * 128);
                    mbar_wait(bar_s + t, g & 1);
                    tc_fence_after();
                    uint32_t sr[128];
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        tmem_ld32(tS + q * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[q * 32]));
                    tmem_ld_wait();
                    tc_fence_before();
                    mbar_arrive(bar_sl + t);  // S_t may be overwritten by the next block's S
                    if (ncols < 128) {  // uniform: the item's last, partial key block
#pragma unroll
                        for (int i = 0; i < 128; ++i)
                            if (i >= ncols) sr[i] = __float_as_uint(-INFINITY);
                    }
                    float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                    for (int i = 0; i < 128; i += 8)
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            mx4[u] = fmax3(mx4[u], __uint_as_float(sr[i + 2 * u]), __uint_as_float(sr[i + 2 * u + 1]));
                    const float mraw = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
                    const float mx = row_ok ? mraw * sl2 : -INFINITY;  // sl2 > 0: max commutes
                    const bool need = mx > m_run + kRescaleThreshold;
                    const float alpha = need ? ex2_approx(m_run - mx) : 1.0f;
                    if (need) {
                        m_run = mx;
                        l_run *= alpha;
                    }
                    const float neg_m = row_ok ? -m_run : -INFINITY;  // dead rows -> p = 0
                    const float2 sl2v = make_float2(sl2, sl2), nm2 = make_float2(neg_m, neg_m);
                    float2 part0 = make_float2(0.f, 0.f), part1 = make_float2(0.f, 0.f);
                    // exponentials by 32-key group; P (bf16 pairs) into this row of the P_t
                    // smem tile, 16-byte chunk q = keys 8q..8q+7 (K-major, 128B swizzle).  The
                    // first two groups are computed before waiting for P_t V of the previous
                    // block (the P_t buffer and O_t), which their exponentials cover.
                    uint32_t pk[32];
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        uint32_t* pg = pk + (cc & 1) * 16;
                        if (cc * 32 >= ncols) {  // uniform: a fully masked group, P = 0
#pragma unroll
                            for (int q = 0; q < 16; ++q) pg[q] = 0u;
                        } else {
#pragma unroll
                            for (int q = 0; q < 16; ++q) {
                                const float2 x = make_float2(__uint_as_float(sr[cc * 32 + 2 * q]),
                                                             __uint_as_float(sr[cc * 32 + 2 * q + 1]));
                                const float2 y = __ffma2_rn(x, sl2v, nm2);
                                float2 e;
                                e.x = ex2_approx(y.x);
                                e.y = ex2_approx(y.y);
                                if (q & 1) part1 = __fadd2_rn(part1, e);
                                else part0 = __fadd2_rn(part0, e);
                                pg[q] = pack_bf16x2(e.x, e.y);
                            }
                        }
                        if (cc == 1 && g > 0) mbar_wait(bar_pv + t, (g - 1) & 1);
                        if (cc & 1) {  // groups cc-1, cc: keys 64 (cc >> 1) .. +64 = strip cc >> 1
                            uint8_t* srow = prow + (cc >> 1) * pstrip;
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                *reinterpret_cast<uint4*>(srow + ((q ^ (row & 7)) << 4)) =
                                    make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                        }
                    }
                    const float2 part = __fadd2_rn(part0, part1);
                    l_run += part.x + part.y;
                    fence_proxy_async_smem();  // st.shared of P -> the MMA's async-proxy reads
                    if (j > 0 && __any_sync(0xffffffffu, need)) {
                        tc_fence_after();
#pragma unroll 1
                        for (int oc = 0; oc < E / 32; ++oc) {
                            uint32_t r[32];
                            tmem_ld32(tO + oc * 32, r);
                            tmem_ld_wait();
#pragma unroll
                            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                            tmem_st32(tO + oc * 32, r);
                        }
                        tmem_st_wait();
                    }
                    tc_fence_before();
                    mbar_arrive(bar_p + t);
                }
                // -------------------------------------------------------- epilogue
                mbar_wait(bar_o + t, li & 1);
                tc_fence_after();
                uint32_t ro[E];
#pragma unroll
                for (int oc = 0; oc < E / 32; ++oc)
                    tmem_ld32(tO + oc * 32, *reinterpret_cast<uint32_t(*)[32]>(&ro[oc * 32]));
                tmem_ld_wait();
                tc_fence_before();  // O reads ordered before this tile's next bar_p arrive
                if (row_ok) {
                    const float inv_l = 1.0f / l_run;
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        uint4 bq[8];
                        if (has_base) {
#pragma unroll
                            for (int q = 0; q < 8; ++q) bq[q] = __ldg(reinterpret_cast<const uint4*>(p.base + off) + hf * 8 + q);
                        }
                        uint4* dp = reinterpret_cast<uint4*>(p.out + off) + hf * 8;
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            float o[8];
#pragma unroll
                            for (int i = 0; i < 8; ++i) o[i] = __uint_as_float(ro[hf * 64 + q * 8 + i]) * inv_l;
                            if (has_base) {
                                const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&bq[q]);
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    const float2 f = __bfloat1622float2(b2[u]);
                                    o[2 * u] = f.x + p.scale * o[2 * u];
                                    o[2 * u + 1] = f.y + p.scale * o[2 * u + 1];
                                }
                            }
                            dp[q] = make_uint4(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]),
                                               pack_bf16x2(o[4], o[5]), pack_bf16x2(o[6], o[7]));
                        }
                    }
                }
                ++li;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

int g_attn_px = [] {
    const char* e = std::getenv("CSD_ATTN_PX");
    return e ? std::atoi(e) : 0;
}();

}  // namespace

bool attn_px_supported(const AttnTcArgs& a) {
    return g_attn_px != 0 && a.idx != nullptr && a.e == E && a.colsum == nullptr && a.row_max == nullptr &&
           a.order == nullptr && a.chunk > 128 && a.chunk <= 192 && a.n % a.chunk == 0;
}

cudaError_t attn_px(const AttnTcArgs& a, cudaStream_t s) {
    const uint64_t cols = a.layout == CSD_LAYOUT_BHNE ? E : (uint64_t)a.heads * E;
    const uint64_t rows = a.layout == CSD_LAYOUT_BHNE ? (uint64_t)(a.batch * a.heads * a.n)
                                                      : (uint64_t)(a.batch * a.n);
    CUtensorMap tq, tb;
    if (!make_map_bf16(&tq, a.q, cols, rows, cols, 64) ||
        !make_map_bf16(&tb, a.base != nullptr ? a.base : a.q, cols, rows, cols, 64))
        return cudaErrorInvalidValue;
    PXParams p{};
    p.idx = a.idx;
    p.counts = a.counts;
    p.k_max = a.k_max;
    p.kp = static_cast<const __nv_bfloat16*>(a.k);
    p.vp = static_cast<const __nv_bfloat16*>(a.v);
    p.base = static_cast<const __nv_bfloat16*>(a.base);
    p.out = static_cast<__nv_bfloat16*>(a.out);
    p.scale = a.scale;
    p.qk_scale_log2 = kLog2e / std::sqrt((float)E);
    p.layout = a.layout;
    p.heads = (int)a.heads;
    p.n = (int)a.n;
    p.chunk = (int)a.chunk;
    p.chunks = (int)(a.n / a.chunk);
    p.items = (int)(a.batch * a.heads * p.chunks);
    p.rows1 = (int)(a.chunk - 128);
    cudaError_t err = ensure_smem_attr(k_attn_px, (int)kSmemBytes);
    if (err != cudaSuccess) return err;
    const unsigned grid = (unsigned)std::min<int64_t>(p.items, sm_count());
    return launch_ex_pdl(1, k_attn_px, dim3(grid), dim3(kThreads), kSmemBytes, s, 1, tq, tb, p);
}

}  // namespace dev
}  // namespace csd

// Debug / test only: route eligible sparse-delta attention launches to the P-in-smem kernel.
extern "C" int csd_debug_set_attn_px(int on) {
    csd::dev::g_attn_px = on;
    return 0;
}
