// attn_sd.cu — dense attention and the dense step's chunk column sums on tcgen05 with a
// DOUBLE-BUFFERED S (CSD_MODE_PROD).
//
// Replaces dense_attention (attention.cpp:59-74) and column_sum_attention (:76-145) for
// head_dim 64 / 128.  Work item = 128 query rows of one (b, h); keys = all N by TMA tiles.
//
// Why a second kernel family next to k_attn_pp: with one M-tile per CTA, TMEM holds two S
// buffers (S(j+1) = Q K_{j+1}^T is computed while the softmax of block j runs, so there is no
// softmax -> P.V -> S chain), O, and the column-sum accumulator:
//   S buffers [0, 256) (P aliased over the first 64 columns of its buffer), O [256, 256+E),
//   D_cs [256+E, 256+E+32) (two 16-column buffers).
// MMA order per key block g: P_g V_g (TS form, A = P from TMEM), then (column sums) D_cs =
// P_g^T W_g, then S_{g+2} into the buffer P_g just left.
//
// Column sums (stale statistics, attention.cpp:122-137): colsum[chunk, key] = sum over the
// chunk's rows r of 2^(s_rk - m_prev_r) / l_prev_r = sum_r w_r p_rk with the online
// probabilities p (already computed) and w_r = 2^(m_run,r - m_prev,r) / l_prev,r.  That is a
// tensor-core product: D_cs[key, n] = sum_r P[r, key] W[r, n], A = P (smem copy, MN-major
// view of the softmax's row-major P), B = W (column 0: w of the rows in the tile's first
// chunk, column 1: the rows of its second chunk).  Four reader warps move D_cs to global
// memory: each (chunk, key) receives at most two fp32 atomic adds onto the zeroed output
// (a 128-row tile meets at most two chunks of 64..256 rows and a chunk at most two tiles),
// so the sums are order-independent and exact in fp32 accumulation.
//
// Roles (16 warps): warp 0 lane 0 Q loader, lane 1 K/V TMA loader; warp 1 MMA issuer;
// warps 4-11 softmax + epilogue (two warps per query-row quadrant, 64 key columns each);
// warps 12-15 column-sum readers.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

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
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;

template <int E>
struct SDLayout {
    static constexpr int kHalves = E / 64;
    static constexpr uint32_t kStrip = 128 * 128;      // 128 rows x 128 B
    static constexpr uint32_t kKV = kHalves * kStrip;  // one K or V block
    static constexpr uint32_t kQ = kHalves * kStrip;
    static constexpr uint32_t kP = 2 * kStrip;         // P copy: 128 rows x 128 keys bf16
    static constexpr uint32_t kW = 2 * 16 * 128;       // W: 16 rows x 128 K, two K strips
    static constexpr uint32_t kThreads = 512;
    static constexpr uint32_t kXch = 2 * 128 * 2 * 4 + 128 * 2 * 4;  // row-half max / sum exchange
    static constexpr uint32_t kOcol = 256;
    static constexpr uint32_t kCscol = 256 + E;
    static constexpr uint32_t kMaxSmem = 227 * 1024;
};

struct SDParams {
    uint32_t off_k, off_v, off_p, off_w, off_x, off_bar;
    int layout, heads, n, tiles, items;  // tiles: 128-row tiles per (b, h)
    __nv_bfloat16* out;
    float* row_max;
    float* exp_sum;
    float* colsum;
    const float* prev_m;
    const float* prev_l;
    int cs_chunk, cs_chunks;
    float qk_scale_log2;
    uint64_t* trace;  // debug timeline (null: off), 8 CTAs x 2048 clock64 stamps
};

#ifdef CSD_SD_NOTRACE  // production builds (paper_2506_03275_b200/build.py; CSD_TRACE=1 keeps it)
#define SD_TRACE(ev, ix) \
    do {                 \
    } while (0)
#else
#define SD_TRACE(ev, ix)                                                                     \
    do {                                                                                     \
        if (p.trace != nullptr && blockIdx.x < 8)                                            \
            p.trace[blockIdx.x * 2048 + (ev) * 64 + ((ix) & 63)] = clock64();                \
    } while (0)
#endif

__device__ __forceinline__ int64_t sd_tok_off(int layout, int64_t b, int64_t h, int64_t tok,
                                              int heads, int n, int e) {
    return layout == CSD_LAYOUT_BHNE ? (((b * heads + h) * (int64_t)n) + tok) * e
                                     : ((b * (int64_t)n + tok) * heads + h) * e;
}

template <int E, int kPoly, bool kCs>
__global__ void __launch_bounds__(SDLayout<E>::kThreads, 1)
k_attn_sd(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
          const __grid_constant__ CUtensorMap tm_v, const SDParams p) {
    using L = SDLayout<E>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_u32 = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int items = p.items;
    const int nblk = (p.n + 127) / 128;  // key blocks per item (every item has all N keys)

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
    uint64_t* bar_q = bars + 0;
    uint64_t* bar_qe = bars + 1;
    uint64_t* bar_kf = bars + 2;   // [2]
    uint64_t* bar_ke = bars + 4;   // [2]
    uint64_t* bar_vf = bars + 6;   // [2]
    uint64_t* bar_ve = bars + 8;   // [2]
    uint64_t* bar_s = bars + 10;   // [2] S buffer b holds S of the current use
    uint64_t* bar_p = bars + 12;   // [2] P_g in TMEM (and the smem copy / W for kCs), by g & 1
    uint64_t* bar_pv = bars + 14;  // P_g V_g completed
    uint64_t* bar_o = bars + 15;   // O final for the item
    uint64_t* bar_cs = bars + 16;  // [2] D_cs buffer full (also: P / W smem consumed)
    uint64_t* bar_csf = bars + 18; // [2] D_cs buffer read out
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);
    uint8_t* const sq = smem;
    uint8_t* const sk = smem + p.off_k;
    uint8_t* const sv = smem + p.off_v;
    uint8_t* const sp = smem + p.off_p;
    uint8_t* const sw = smem + p.off_w;
    float* const xch = reinterpret_cast<float*>(smem + p.off_x);       // [2][128][2] block maxima
    float* const lxch = xch + 2 * 128 * 2;                              // [128][2] row sums
    if (threadIdx.x == 0) {
        if ((raw_u32 & 1023u) != 0) __trap();
        mbar_init(bar_q, 1);
        mbar_init(bar_qe, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar_kf + i, 1);
            mbar_init(bar_ke + i, 1);
            mbar_init(bar_vf + i, 1);
            mbar_init(bar_ve + i, 1);
            mbar_init(bar_s + i, 1);
            mbar_init(bar_cs + i, 1);
            mbar_init(bar_csf + i, 128);
            mbar_init(bar_p + i, 256);  // both row halves
        }
        mbar_init(bar_pv, 1);
        mbar_init(bar_o, 1);
        fence_barrier_init();
    }
    if (kCs) {  // W rows 2..15 stay zero
        for (uint32_t i = threadIdx.x; i < L::kW / 16; i += blockDim.x)
            reinterpret_cast<uint4*>(sw)[i] = make_uint4(0u, 0u, 0u, 0u);
        fence_proxy_async_smem();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    if (threadIdx.x == 0) pdl_trigger();
    auto item_rows = [&](int it, int& q_row, int& k_row, int& col0) {
        const int bh = it / p.tiles;
        k_row = p.layout == CSD_LAYOUT_BHNE ? bh * p.n : (bh / p.heads) * p.n;
        col0 = p.layout == CSD_LAYOUT_BHNE ? 0 : (bh % p.heads) * E;
        q_row = k_row + (it % p.tiles) * 128;
    };

    // registers: 8 softmax warps at 168, the 8 others at 88 (512 threads x 128 at launch)
    if (warp < 4) {
        regs_dec<88>();
        if (warp == 0 && lane == 0) {
            // ---------------------------------------------------------- Q loader
            tma_prefetch_desc(&tm_q);
            uint32_t li = 0;
            for (int it = blockIdx.x; it < items; it += gridDim.x, ++li) {
                int qr, kr, col0;
                item_rows(it, qr, kr, col0);
                if (li > 0) mbar_wait(bar_qe, (li - 1) & 1);
                mbar_arrive_expect_tx(bar_q, L::kQ);
                for (int hf = 0; hf < L::kHalves; ++hf)
                    for (int bx = 0; bx < 2; ++bx)
                        tma_load_2d(&tm_q, bar_q, sq + hf * L::kStrip + bx * 8192, col0 + hf * 64, qr + bx * 64);
                if (it + (int)gridDim.x < items) {
                    int nqr, nkr, ncol0;
                    item_rows(it + gridDim.x, nqr, nkr, ncol0);
                    for (int hf = 0; hf < L::kHalves; ++hf)
                        for (int bx = 0; bx < 2; ++bx) tma_prefetch_2d(&tm_q, ncol0 + hf * 64, nqr + bx * 64);
                }
            }
        } else if (warp == 2 && lane == 0) {  // own warp: a divergent lane of warp 0 waits behind the Q loader's spins
            // ---------------------------------------------------------- K / V TMA tiles
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_v);
            uint32_t g = 0;
            for (int it = blockIdx.x; it < items; it += gridDim.x) {
                int qr, kr, col0;
                item_rows(it, qr, kr, col0);
                for (int j = 0; j < nblk; ++j, ++g) {
                    const int s = g & 1;
                    if (g >= 2) mbar_wait(bar_ke + s, ((g >> 1) - 1) & 1);
                    mbar_arrive_expect_tx(bar_kf + s, L::kKV);
                    for (int hf = 0; hf < L::kHalves; ++hf)
                        tma_load_2d(&tm_k, bar_kf + s, sk + s * L::kKV + hf * L::kStrip, col0 + hf * 64, kr + j * 128);
                    if (g >= 2) mbar_wait(bar_ve + s, ((g >> 1) - 1) & 1);
                    mbar_arrive_expect_tx(bar_vf + s, L::kKV);
                    for (int hf = 0; hf < L::kHalves; ++hf)
                        tma_load_2d(&tm_v, bar_vf + s, sv + s * L::kKV + hf * L::kStrip, col0 + hf * 64, kr + j * 128);
                }
            }
        } else if (warp == 1) {
            // ---------------------------------------------------------- MMA issuer
            constexpr uint32_t idS = idesc_bf16(128, 128, false, false);
            constexpr uint32_t idO = idesc_bf16(128, E, false, true);
            constexpr uint32_t idC = idesc_bf16(128, 16, true, false);
            const uint32_t sQ = smem_u32(sq), sK = smem_u32(sk), sV = smem_u32(sv);
            const uint32_t sP = smem_u32(sp), sW = smem_u32(sw);
            auto commit = [&](uint64_t* b) {
                if (elect_one()) mma_commit(b);
                __syncwarp();
            };
            auto issue_s = [&](uint32_t g) {  // S buffer g & 1 = Q K_g^T
                const uint32_t kb = sK + (g & 1) * L::kKV;
                uint64_t da[E / 16], db[E / 16];
#pragma unroll
                for (int kk = 0; kk < E / 16; ++kk) {
                    da[kk] = desc_kmajor_sw128(sQ + (kk / 4) * L::kStrip + (kk % 4) * 32);
                    db[kk] = desc_kmajor_sw128(kb + (kk / 4) * L::kStrip + (kk % 4) * 32);
                }
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < E / 16; ++kk)
                        mma_bf16(tmem + (g & 1) * 128, da[kk], db[kk], idS, kk > 0 ? 1u : 0u);
                    mma_commit(bar_s + (g & 1));
                    mma_commit(bar_ke + (g & 1));
                }
                __syncwarp();
            };
            const int total = ((items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * nblk;
            // block g -> (local item li = g / nblk, j = g % nblk); S of block g needs Q of its item
            uint32_t q_have = 0;  // Q of local items < q_have has been waited for
            auto want_q = [&](uint32_t g) {
                const uint32_t li = g / nblk;
                if (li + 1 > q_have) {
                    mbar_wait(bar_q, li & 1);
                    q_have = li + 1;
                }
            };
            auto s_block = [&](uint32_t g) {  // issue S of block g (and release Q after the item's last)
                want_q(g);
                mbar_wait(bar_kf + (g & 1), (g >> 1) & 1);
                tc_fence_after();
                if (lane == 0) SD_TRACE(0, g);
                issue_s(g);
                if ((int)(g % nblk) == nblk - 1) commit(bar_qe);
            };
            if (total > 0) s_block(0);
            if (total > 1) s_block(1);
            for (uint32_t g = 0; (int)g < total; ++g) {
                const int j = (int)(g % nblk);
                mbar_wait(bar_p + (g & 1), (g >> 1) & 1);
                if (lane == 0) SD_TRACE(1, g);
                mbar_wait(bar_vf + (g & 1), (g >> 1) & 1);
                tc_fence_after();
                {
                    const uint32_t vb = sV + (g & 1) * L::kKV;
                    uint64_t dv[8];
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) dv[kk] = desc_mnmajor_sw128(vb + kk * 2048, L::kStrip);
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)
                            mma_bf16_ts(tmem + L::kOcol, tmem + (g & 1) * 128 + kk * 8, dv[kk], idO,
                                        (j > 0 || kk > 0) ? 1u : 0u);
                        mma_commit(bar_ve + (g & 1));
                        mma_commit(bar_pv);
                        if (j == nblk - 1) mma_commit(bar_o);
                    }
                    __syncwarp();
                }
                if (kCs) {
                    // D_cs[g & 1] = P_g^T W_g (keys x 16)
                    if (g >= 2) mbar_wait(bar_csf + (g & 1), ((g >> 1) - 1) & 1);
                    tc_fence_after();
                    uint64_t da[8], db[8];
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        da[kk] = desc_mnmajor_sw128(sP + kk * 2048, L::kStrip);
                        db[kk] = desc_kmajor_sw128(sW + (kk / 4) * 2048 + (kk % 4) * 32);
                    }
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)
                            mma_bf16(tmem + L::kCscol + (g & 1) * 16, da[kk], db[kk], idC, kk > 0 ? 1u : 0u);
                        mma_commit(bar_cs + (g & 1));
                    }
                    __syncwarp();
                }
                if ((int)g + 2 < total) s_block(g + 2);  // into the buffer P_g just left
            }
        }
    } else if (warp < 12) {
        regs_inc<168>();
        // -------------------------------------------------------------- softmax + epilogue
        // two warps per TMEM lane quadrant (warps 4 + q and 8 + q, both on SMSP q): half h
        // owns key columns [64 h, 64 h + 64) of every block and O columns [E/2 h, E/2 h + E/2);
        // the halves swap their block maxima through shared memory (64-thread named barrier
        // per quadrant) and their row sums once per item
        const int quad = warp & 3, hf = (warp - 4) >> 2;
        const int row = quad * 32 + lane;
        const uint32_t bar_id = 1 + quad;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const uint32_t tO = tmem + lane_off + L::kOcol + hf * (E / 2);
        const float sl2 = p.qk_scale_log2;
        uint32_t g = 0, li = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x, ++li) {
            const int bh = it / p.tiles, b = bh / p.heads, h = bh % p.heads;
            const int64_t tok = (int64_t)(it % p.tiles) * 128 + row;
            const bool row_ok = tok < p.n;
            float m_run = -INFINITY, m_true = -INFINITY, l_run = 0.f;
            float mpl = 0.f, inv_lp = 0.f;
            int slot = 0;  // kCs: W column of this row's chunk (0: the tile's first chunk)
            if (kCs && row_ok) {
                const int64_t si = (int64_t)bh * p.n + tok;
                mpl = p.prev_m[si] * kLog2e;
                inv_lp = 1.0f / p.prev_l[si];
                slot = (int)(tok / p.cs_chunk - ((int64_t)(it % p.tiles) * 128) / p.cs_chunk);
            }
            for (int j = 0; j < nblk; ++j, ++g) {
                const int nh = min(64, max(0, p.n - j * 128 - 64 * hf));  // live columns of this half
                const uint32_t tS = tmem + lane_off + (g & 1) * 128;
                mbar_wait(bar_s + (g & 1), (g >> 1) & 1);
                tc_fence_after();
                if (lane == 0 && warp == 4) SD_TRACE(2, g);
                if (lane == 0 && warp == 8) SD_TRACE(3, g);
                uint32_t sr[64];
                tmem_ld32(tS + hf * 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
                tmem_ld32(tS + hf * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
                tmem_ld_wait();
                if (nh < 64) {
#pragma unroll
                    for (int i = 0; i < 64; ++i)
                        if (i >= nh) sr[i] = __float_as_uint(-INFINITY);
                }
                float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int i = 0; i < 64; i += 8)
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        mx4[u] = fmax3(mx4[u], __uint_as_float(sr[i + 2 * u]), __uint_as_float(sr[i + 2 * u + 1]));
                const float mloc = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
                float* xr = xch + ((g & 1) * 128 + row) * 2;
                xr[hf] = mloc;
                named_bar_sync(bar_id, 64);
                const float mraw = fmaxf(mloc, xr[hf ^ 1]);
                if (lane == 0 && warp == 4) SD_TRACE(6, g);
                const float mx = row_ok ? mraw * sl2 : -INFINITY;
                m_true = fmaxf(m_true, mx);
                const bool need = mx > m_run + kRescaleThreshold;
                const float alpha = need ? ex2_approx(m_run - mx) : 1.0f;
                if (need) {
                    m_run = mx;
                    l_run *= alpha;
                }
                const float neg_m = row_ok ? -m_run : -INFINITY;
                const float2 sl2v = make_float2(sl2, sl2), nm2 = make_float2(neg_m, neg_m);
                float2 part0 = make_float2(0.f, 0.f), part1 = make_float2(0.f, 0.f);
                // P of both 32-key groups stays in registers until the smem copy (kCs): the
                // wait for the previous block's column-sum MMA (P / W smem free) comes after the
                // exponentials instead of before them
                uint32_t pka[32];
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    uint32_t(&pk)[16] = *reinterpret_cast<uint32_t(*)[16]>(&pka[cc * 16]);
                    if (cc * 32 >= nh) {
#pragma unroll
                        for (int q = 0; q < 16; ++q) pk[q] = 0u;
                    } else {
#pragma unroll
                        for (int q = 0; q < 16; ++q) {
                            const float2 x = make_float2(__uint_as_float(sr[cc * 32 + 2 * q]),
                                                         __uint_as_float(sr[cc * 32 + 2 * q + 1]));
                            const float2 y = __ffma2_rn(x, sl2v, nm2);
                            float2 e;
                            if (kPoly > 0 && (q % (kPoly > 0 ? kPoly : 1)) == kPoly - 1) {
                                e = ex2_poly2(y);
                            } else {
                                e.x = ex2_approx(y.x);
                                e.y = ex2_approx(y.y);
                            }
                            if (q & 1) part1 = __fadd2_rn(part1, e);
                            else part0 = __fadd2_rn(part0, e);
                            pk[q] = pack_bf16x2(e.x, e.y);
                        }
                    }
                    tmem_st16(tS + hf * 32 + cc * 16, pk);  // P of keys 64 hf + 32 cc ..
                }
                const float2 part = __fadd2_rn(part0, part1);
                l_run += part.x + part.y;
                if (kCs) {
                    if (g >= 1) mbar_wait(bar_cs + ((g - 1) & 1), ((g - 1) >> 1) & 1);  // P/W smem free
                    // the row's P copy (K-major, 128B-swizzled): strip hf, 16-byte chunks 0..7
                    uint8_t* rp = sp + hf * L::kStrip + row * 128;
#pragma unroll
                    for (int ch = 0; ch < 8; ++ch)
                        *reinterpret_cast<uint4*>(rp + ((ch ^ (row & 7)) << 4)) =
                            make_uint4(pka[4 * ch], pka[4 * ch + 1], pka[4 * ch + 2], pka[4 * ch + 3]);
                    if (hf == 0) {
                        // W[slot][row] = w, W[1 - slot][row] = 0 (bf16, K-major 128B-swizzled).
                        // Stale stats far below the fresh logits: the reference's fp32 exp
                        // overflows to +inf past ~88 nats (attention.cpp:135); a finite cap keeps
                        // those products overflowing (p w -> +inf in the MMA) without turning the
                        // masked p = 0 entries into inf * 0 = NaN
                        const float w = row_ok ? fminf(ex2_approx(m_run - mpl) * inv_lp, 3.0e38f) : 0.f;
                        const __nv_bfloat16 wb = __float2bfloat16_rn(w), zb = __float2bfloat16_rn(0.f);
                        uint8_t* ws = sw + (row >> 6) * 2048;
                        const int kc = (row & 63) >> 3, ke = row & 7;
#pragma unroll
                        for (int n = 0; n < 2; ++n)
                            *reinterpret_cast<__nv_bfloat16*>(ws + n * 128 + (((kc ^ n) & 7) << 4) + ke * 2) =
                                n == slot ? wb : zb;
                    }
                    fence_proxy_async_smem();  // generic smem writes -> the MMA's async proxy
                }
                if (j > 0 && __any_sync(0xffffffffu, need)) {
                    // O holds P V of blocks < j once P_{g-1} V_{g-1} completed; this half's columns
                    mbar_wait(bar_pv, (g - 1) & 1);
                    tc_fence_after();
#pragma unroll 1
                    for (int oc = 0; oc < E / 64; ++oc) {
                        uint32_t r[32];
                        tmem_ld32(tO + oc * 32, r);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                        tmem_st32(tO + oc * 32, r);
                    }
                }
                tmem_st_wait();
                tc_fence_before();
                if (lane == 0 && warp == 4) SD_TRACE(4, g);
                if (lane == 0 && warp == 8) SD_TRACE(5, g);
                mbar_arrive(bar_p + (g & 1));
            }
            // ------------------------------------------------------------ epilogue
            lxch[row * 2 + hf] = l_run;
            named_bar_sync(bar_id, 64);
            const float l_full = l_run + lxch[row * 2 + (hf ^ 1)];
            mbar_wait(bar_o, li & 1);
            tc_fence_after();
            {
                uint32_t ro[E / 2];
#pragma unroll
                for (int oc = 0; oc < E / 64; ++oc)
                    tmem_ld32(tO + oc * 32, *reinterpret_cast<uint32_t(*)[32]>(&ro[oc * 32]));
                tmem_ld_wait();
                if (row_ok) {
                    const float inv_l = 1.0f / l_full;
                    uint4* dp = reinterpret_cast<uint4*>(p.out + sd_tok_off(p.layout, b, h, tok, p.heads, p.n, E) +
                                                         hf * (E / 2));
#pragma unroll
                    for (int q = 0; q < E / 16; ++q)
                        dp[q] = make_uint4(pack_bf16x2(__uint_as_float(ro[8 * q]) * inv_l, __uint_as_float(ro[8 * q + 1]) * inv_l),
                                           pack_bf16x2(__uint_as_float(ro[8 * q + 2]) * inv_l, __uint_as_float(ro[8 * q + 3]) * inv_l),
                                           pack_bf16x2(__uint_as_float(ro[8 * q + 4]) * inv_l, __uint_as_float(ro[8 * q + 5]) * inv_l),
                                           pack_bf16x2(__uint_as_float(ro[8 * q + 6]) * inv_l, __uint_as_float(ro[8 * q + 7]) * inv_l));
                    if (hf == 0 && p.row_max != nullptr) {
                        const int64_t si = (int64_t)bh * p.n + tok;
                        p.row_max[si] = m_true * kLn2;
                        p.exp_sum[si] = l_full * exp2f(m_run - m_true);
                    }
                }
            }
            named_bar_sync(bar_id, 64);  // lxch read by both halves before the next item's write
            tc_fence_before();  // O reads ordered before the next item's first bar_p arrive
        }
    } else {
        regs_dec<88>();
        if (kCs) {
            // ---------------------------------------------------------- column-sum readers
            const int quad = warp - 12;
            const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
            uint32_t g = 0;
            for (int it = blockIdx.x; it < items; it += gridDim.x) {
                const int bh = it / p.tiles;
                const int64_t r0 = (int64_t)(it % p.tiles) * 128;
                const int64_t c_lo = r0 / p.cs_chunk;
                const int64_t r_last = std::min<int64_t>(r0 + 127, p.n - 1);
                const bool two = r_last / p.cs_chunk != c_lo;
                float* dst0 = p.colsum + ((int64_t)bh * p.cs_chunks + c_lo) * p.n;
                for (int j = 0; j < nblk; ++j, ++g) {
                    mbar_wait(bar_cs + (g & 1), (g >> 1) & 1);
                    tc_fence_after();
                    uint32_t v[2];
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                                 : "=r"(v[0]), "=r"(v[1])
                                 : "r"(tmem + lane_off + L::kCscol + (g & 1) * 16));
                    tmem_ld_wait();
                    tc_fence_before();
                    mbar_arrive(bar_csf + (g & 1));
                    const int key = j * 128 + quad * 32 + lane;
                    if (key < p.n) {
                        atomicAdd(dst0 + key, __uint_as_float(v[0]));
                        if (two) atomicAdd(dst0 + p.n + key, __uint_as_float(v[1]));
                    }
                }
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

uint64_t* h_sd_trace = nullptr;

template <int E>
cudaError_t launch_sd(const AttnTcArgs& a, cudaStream_t s) {
    using L = SDLayout<E>;
    const uint64_t cols = a.layout == CSD_LAYOUT_BHNE ? E : (uint64_t)a.heads * E;
    const uint64_t rows = a.layout == CSD_LAYOUT_BHNE ? (uint64_t)(a.batch * a.heads * a.n)
                                                      : (uint64_t)(a.batch * a.n);
    CUtensorMap tq, tk, tv;
    if (!make_map_bf16(&tq, a.q, cols, rows, cols, 64) || !make_map_bf16(&tk, a.k, cols, rows, cols, 128) ||
        !make_map_bf16(&tv, a.v, cols, rows, cols, 128))
        return cudaErrorInvalidValue;
    SDParams p{};
    p.layout = a.layout;
    p.heads = (int)a.heads;
    p.n = (int)a.n;
    p.tiles = (int)((a.n + 127) / 128);
    p.items = (int)(a.batch * a.heads * p.tiles);
    p.out = static_cast<__nv_bfloat16*>(a.out);
    p.row_max = a.row_max;
    p.exp_sum = a.exp_sum;
    p.qk_scale_log2 = kLog2e / std::sqrt((float)E);
    p.trace = h_sd_trace;
    const bool cs = a.colsum != nullptr;
    uint32_t off = L::kQ;
    p.off_k = off;
    p.off_v = off + 2 * L::kKV;
    off = p.off_v + 2 * L::kKV;
    p.off_p = off;
    p.off_w = off + (cs ? L::kP : 0);
    p.off_x = p.off_w + (cs ? L::kW : 0);
    p.off_bar = p.off_x + L::kXch;
    const uint32_t smem_bytes = p.off_bar + 256;
    if (smem_bytes > L::kMaxSmem) return cudaErrorNotSupported;
    if (cs) {
        p.colsum = a.colsum;
        p.prev_m = a.prev_m;
        p.prev_l = a.prev_l;
        p.cs_chunk = a.cs_chunk > 0 ? (int)a.cs_chunk : (int)a.chunk;
        p.cs_chunks = (int)(a.n / p.cs_chunk);
        cudaError_t e = cudaMemsetAsync(a.colsum, 0, sizeof(float) * a.batch * a.heads * p.cs_chunks * a.n, s);
        if (e != cudaSuccess) return e;
    }
    static const int poly_env = [] {
        const char* e = std::getenv("CSD_SD_POLY");
        return e ? std::atoi(e) : -1;
    }();
    const int poly = poly_env >= 0 ? poly_env : 0;
    auto kern = cs ? (poly == 4 ? k_attn_sd<E, 4, true> : k_attn_sd<E, 0, true>)
                   : (poly == 4 ? k_attn_sd<E, 4, false> : k_attn_sd<E, 0, false>);
    cudaError_t err = ensure_smem_attr(kern, (int)L::kMaxSmem);
    if (err != cudaSuccess) return err;
    const unsigned grid = (unsigned)std::min<int64_t>(p.items, sm_count());
    return launch_ex(kern, dim3(grid), dim3(L::kThreads), smem_bytes, s, 1, tq, tk, tv, p);
}

}  // namespace

// Dense passes (no index set, no base): plain dense attention, the dense step's stats pass and
// its column-sum pass.  CSD_ATTN_DENSE=pp|tc keeps them on the other kernels.
bool attn_sd_supported(const AttnTcArgs& a) {
    static const int mode = [] {
        const char* e = std::getenv("CSD_ATTN_DENSE");
        return e == nullptr ? 0 : std::string(e) == "pp" ? 1 : std::string(e) == "tc" ? 2 : 0;
    }();
    if (mode != 0 || a.idx != nullptr || a.base != nullptr || !(a.e == 64 || a.e == 128)) return false;
    if (a.colsum == nullptr) return true;
    const int64_t cs = a.cs_chunk > 0 ? a.cs_chunk : a.chunk;
    return a.prev_m != nullptr && a.prev_l != nullptr && a.n % cs == 0 &&
           (cs == 64 || cs == 128 || cs == 192 || cs == 256);
}

cudaError_t attn_sd(const AttnTcArgs& a, cudaStream_t s) {
    return a.e == 128 ? launch_sd<128>(a, s) : launch_sd<64>(a, s);
}

}  // namespace dev
}  // namespace csd

// Debug only: clock64 timeline of k_attn_sd's first 8 CTAs (8 x 2048 uint64; null: off).
extern "C" int csd_debug_set_attn_sd_trace(void* dev_buf) {
    csd::dev::h_sd_trace = static_cast<uint64_t*>(dev_buf);
    return 0;
}
