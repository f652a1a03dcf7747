// attn_pp.cu — column-sparse / dense attention with ping-pong M-tiles (CSD_MODE_PROD).
//
// Replaces sparse_delta_attention (attention.cpp:147-194) and dense_attention (:59-74) for
// work items of 129..256 query rows (FLUX / Hunyuan chunk 192; dense passes use 256-row
// items).  The dense-step column sums (:76-145) stay in attn_tc.cu.
//
// Work item = (b, h, query chunk): two M-tiles of 128 rows that share every K/V block
// (tile 1 holds rows 128..chunk-1).  Unlike k_attn_tc, each tile has its OWN softmax
// warpgroup (4 warps, one thread per query row holding all 128 key columns of the block)
// and its own Q / S / P / O barriers, so the per-tile chain
//     softmax_t(j) -> P_t V_j -> S_t(j+1) = Q_t K_{j+1}^T -> softmax_t(j+1)
// of one tile overlaps the other tile's MMAs and softmax, and it continues ACROSS items:
// the MMA warp walks one flattened key-block sequence over all items of its CTA, issuing
// the next item's first S as soon as that tile's Q is in (Q tiles are released per tile as
// soon as their last S MMA completes, and the next item's Q is L2-prefetched when the
// current one is loaded).  The epilogue (out = base + scale * O / l, north_star item 5) is
// run by each tile's softmax warpgroup while the MMA pipe already computes the next item's
// first S blocks.
//
// TMEM (512 columns): S_0 [0,128), S_1 [128,256) (P_t aliased over the first 64 columns of
// S_t as bf16 pairs), O_0 [256, 256+E), O_1 [256+E, 256+2E).
//
// Roles (16 warps): warp 0 lane 0 Q loader; warp 1 MMA issuer; warp 2 lane 0 dense K/V TMA
// loader (dense passes) or, with warps 12-15, the sparse K/V row copies (cp.async); warp 3
// lane 0 staged-base / out I/O; warps 4-7 softmax tile 0; warps 8-11 softmax tile 1.  (Each
// single-thread role has its own warp: divergent lanes of one warp delay each other's
// barrier waits.)
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
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale only when the max grows > 2^8

template <int E>
struct PPLayout {
    static constexpr int kHalves = E / 64;
    static constexpr uint32_t kStrip = 128 * 128;      // 128 rows x 128 B
    static constexpr uint32_t kKV = kHalves * kStrip;  // one K or V block
    static constexpr uint32_t kThreads = 512;
    static constexpr int kCopyThreads = 160;  // warps 2, 12-15 (warp 3: staged base / out I/O)
    static constexpr uint32_t kTmemCols = 512;
    static constexpr uint32_t kOcol = 256;    // O_0 column
    static constexpr uint32_t kMaxSmem = 227 * 1024;
};

struct PPParams {
    int stage_base;               // base tile staged in smem region X (epilogue in smem)
    uint32_t off_q[2], q_strip[2];  // per M-tile: Q region offset, bytes per 64-column strip
    int q_rows[2];                // per M-tile: Q rows loaded (multiple of 64)
    int rows[2];                  // per M-tile: live query rows
    uint32_t off_x, x_strip, off_k, off_v, off_bar;
    const int32_t* idx;
    const int32_t* counts;
    int64_t k_max;
    const __nv_bfloat16* base;
    __nv_bfloat16* out;
    float scale;
    float* row_max;
    float* exp_sum;
    int layout;
    int heads, n, chunk, chunks, items;
    const __nv_bfloat16* kp;
    const __nv_bfloat16* vp;
    float qk_scale_log2;
    int warm;  // dead softmax warps run the first item as an icache warm-up (softmax branch)
    const int32_t* order;  // work position -> item (longest first), or null (identity)
    uint64_t* span;  // debug per-CTA [start, end] globaltimer (null: off)
    uint64_t* trace;  // debug timeline (null: off): kPPTraceCtas x 1024 clock64 stamps
};

// Debug timeline (scripts/attn_pp_trace.py): CTAs < kPPTraceCtas stamp clock64() at slot (of 2048)
// event * 64 + (index & 63); the pointer travels in the parameters (constant bank).
constexpr int kPPTraceCtas = 8;
#ifdef CSD_PP_NOTRACE
#define PP_TRACE(ev, ix) \
    do {                 \
    } while (0)
#else
#define PP_TRACE(ev, ix)                                                                     \
    do {                                                                                     \
        if (p.trace != nullptr && blockIdx.x < kPPTraceCtas)                                 \
            p.trace[blockIdx.x * 2048 + (ev) * 64 + ((ix) & 63)] = clock64();                \
    } while (0)
#endif

__device__ __forceinline__ int64_t pp_tok_off(int layout, int64_t b, int64_t h, int64_t tok,
                                              int heads, int n, int e) {
    return layout == CSD_LAYOUT_BHNE ? (((b * heads + h) * (int64_t)n) + tok) * e
                                     : ((b * (int64_t)n + tok) * heads + h) * e;
}

// predicated 16-byte stores (the dry warm-up pass runs the epilogue code without storing;
// inline PTX keeps the compiler from unswitching the loop into a second, store-free copy)
__device__ __forceinline__ void st_shared_v4_if(bool on, void* ptr, const uint32_t (&v)[4]) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %5, 0;\n @p st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n}"
                 ::"r"(smem_u32(ptr)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"((int)on)
                 : "memory");
}
__device__ __forceinline__ void st_global_v4_if(bool on, void* ptr, const uint4& v) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %5, 0;\n @p st.global.v4.b32 [%0], {%1, %2, %3, %4};\n}"
                 ::"l"(ptr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"((int)on)
                 : "memory");
}

__device__ __forceinline__ uint64_t pp_globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// kPoly > 0: every kPoly-th exponential pair of a row runs as a degree-3 polynomial on the
// FMA pipe instead of MUFU (ex2_poly2), balancing the two pipes.
// kOrd: the launch carries an LPT item order (p.order).  Without it the order indirection is
// compiled out: a kernel-wide order pointer is otherwise spilled (128-register launch bound)
// and reloaded from local memory at every item lookup.
// kDense: dense passes (all keys by TMA tiles) vs sparse items (gathered K/V rows); a
// compile-time split so each instance carries only its own code (instruction fetch is a
// measured cost of this kernel: the cold first item after the Q/K/V GEMM)
template <int E, int kPoly, bool kOrd, bool kDense>
__global__ void __launch_bounds__(PPLayout<E>::kThreads, 1)
k_attn_pp(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
          const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_b,
          const __grid_constant__ CUtensorMap tm_o, const PPParams p) {
    using L = PPLayout<E>;
    static_assert(kPoly == 0 || kPoly >= 2, "poly split");
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_u32 = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr bool dense = kDense;
    const int items = p.items;
    if (threadIdx.x == 0 && p.span != nullptr) p.span[2 * blockIdx.x] = pp_globaltimer();
    if (threadIdx.x == 0) PP_TRACE(15, 0);

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
    uint64_t* bar_q = bars + 0;    // [2] Q tile t landed
    uint64_t* bar_qe = bars + 2;   // [2] Q tile t free (the item's last S_t MMA completed)
    uint64_t* bar_kf = bars + 4;   // [2] K ring slot full
    uint64_t* bar_ke = bars + 6;   // [2] K ring slot free
    uint64_t* bar_vf = bars + 8;   // [2]
    uint64_t* bar_ve = bars + 10;  // [2]
    uint64_t* bar_s = bars + 12;   // [2] S_t in TMEM
    uint64_t* bar_p = bars + 14;   // [2] P_t in TMEM (and O_t rescaled / read out)
    uint64_t* bar_o = bars + 16;   // [2] O_t final for the item
    uint64_t* bar_bf = bars + 18;  // staged base tile of the current live item landed
    uint64_t* bar_xc = bars + 19;  // every live softmax warp combined its rows into X
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);
    uint8_t* const sx = smem + p.off_x;
    uint8_t* const sk = smem + p.off_k;
    uint8_t* const sv = smem + p.off_v;
    const int lw0 = (p.rows[0] + 31) >> 5, lw1 = (p.rows[1] + 31) >> 5;  // live warps per tile
    const bool cpa = !dense;
    if (threadIdx.x == 0) {
        if ((raw_u32 & 1023u) != 0) __trap();  // the host sizes the request without slack
        const uint32_t fill = cpa ? (uint32_t)L::kCopyThreads : 1u;
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar_q + i, 1);
            mbar_init(bar_qe + i, 1);
            mbar_init(bar_kf + i, fill);
            mbar_init(bar_ke + i, 1);
            mbar_init(bar_vf + i, fill);
            mbar_init(bar_ve + i, 1);
            mbar_init(bar_s + i, 1);
            mbar_init(bar_o + i, 1);
        }
        mbar_init(bar_p + 0, 32u * lw0);
        mbar_init(bar_p + 1, 32u * lw1);
        mbar_init(bar_bf, 1);
        mbar_init(bar_xc, (uint32_t)(lw0 + lw1));
        fence_barrier_init();
    }
    // work positions -> items: longest-first order for ragged index sets (p.order, LPT), or
    // the identity; every role walks POSITIONS pos = blockIdx.x + i * gridDim.x
    const int32_t* order = (kOrd && p.order[items] == 0) ? p.order : nullptr;
    // (captured by value: a by-reference capture gives `order` a stack slot that every
    // asm "memory" clobber then reloads -- LDL on the hot paths)
    auto item_at = [order](int pos) -> int { return order != nullptr ? order[pos] : pos; };
    auto count_of = [=](int pos) -> int { return dense ? p.n : p.counts[item_at(pos)]; };
    // next live (count > 0) item of this CTA at or after `from`
    auto next_live = [=](int from, int& cnt_out) -> int {
        int x = from;
        cnt_out = 0;
        for (; x < items; x += gridDim.x) {
            cnt_out = count_of(x);
            if (cnt_out > 0) break;
        }
        return x;
    };
    auto item_rows = [=](int pos, int& row_base, int& col0) {
        const int it = item_at(pos);
        const int bh = it / p.chunks;
        row_base = p.layout == CSD_LAYOUT_BHNE ? bh * p.n : (bh / p.heads) * p.n;
        col0 = p.layout == CSD_LAYOUT_BHNE ? 0 : (bh % p.heads) * E;
        row_base += (it % p.chunks) * p.chunk;
    };

    // sparse K/V copy threads: their first item's count and first block's indices are
    // loaded before the setup barrier (the DRAM latency overlaps the TMEM allocation)
    static_assert(L::kCopyThreads % (E / 8) == 0, "copy threads per row");
    constexpr int kRowStep = L::kCopyThreads / (E / 8);
    constexpr int kCpRows = (128 + kRowStep - 1) / kRowStep;
    const int cp_thread = warp == 2 ? lane : 32 + (warp - 12) * 32 + lane;
    auto load_ids = [=](int it, int cnt, int j, int32_t (&id)[kCpRows]) {
        const int r0 = cp_thread / (E / 8);
        const int32_t* ids = p.idx + (int64_t)(it < items ? item_at(it) : 0) * p.k_max;
#pragma unroll
        for (int i = 0; i < kCpRows; ++i) {
            const int r = j * 128 + r0 + kRowStep * i;
            id[i] = (it < items && r0 + kRowStep * i < 128 && r < cnt) ? __ldg(ids + r) : -1;
        }
    };
    int cp_it = items, cp_cnt = 0;
    int32_t cp_id[kCpRows];
    if (cpa && (warp == 2 || warp >= 12)) {
        pdl_wait();  // the counts / indices may come from the previous kernel (dense step top-k)
        cp_it = next_live(blockIdx.x, cp_cnt);
        load_ids(cp_it, cp_cnt, 0, cp_id);
    }
    if (warp == 1) tmem_alloc<L::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 4 || warp >= 12) {
        regs_dec<72>();
        pdl_wait();
        if (threadIdx.x == 0) pdl_trigger();
        if (warp == 0) {
            if (lane == 0) {
                // ---------------------------------------------------- Q loader (per tile)
                tma_prefetch_desc(&tm_q);
                uint32_t li = 0;
                int cnt = 0;
                for (int it = next_live(blockIdx.x, cnt); it < items; ++li) {
                    int r0, col0;
                    item_rows(it, r0, col0);
                    for (int t = 0; t < 2; ++t) {
                        if (li > 0) mbar_wait(bar_qe + t, (li - 1) & 1);
                        PP_TRACE(13 + t, li);
                        mbar_arrive_expect_tx(bar_q + t, (uint32_t)(L::kHalves * p.q_rows[t]) * 128u);
                        for (int hf = 0; hf < L::kHalves; ++hf)
                            for (int bx = 0; bx < p.q_rows[t] / 64; ++bx)
                                tma_load_2d(&tm_q, bar_q + t,
                                            smem + p.off_q[t] + hf * p.q_strip[t] + bx * 8192,
                                            col0 + hf * 64, r0 + t * 128 + bx * 64);
                    }
                    const int nx = next_live(it + gridDim.x, cnt);
                    if (nx < items) {  // the next item's Q into L2 while this one runs
                        int nr0, ncol0;
                        item_rows(nx, nr0, ncol0);
                        for (int t = 0; t < 2; ++t)
                            for (int hf = 0; hf < L::kHalves; ++hf)
                                for (int bx = 0; bx < p.q_rows[t] / 64; ++bx)
                                    tma_prefetch_2d(&tm_q, ncol0 + hf * 64, nr0 + t * 128 + bx * 64);
                    }
                    it = nx;
                }
            }
        } else if (warp == 2 && dense) {  // own warp (a divergent lane of warp 0 waits behind its spins)
            if (lane == 0) {
                // ---------------------------------------------------- dense K/V TMA tiles
                tma_prefetch_desc(&tm_k);
                tma_prefetch_desc(&tm_v);
                uint32_t gb = 0;
                int cnt = 0;
                for (int it = next_live(blockIdx.x, cnt); it < items; it = next_live(it + gridDim.x, cnt)) {
                    int r0, col0;
                    item_rows(it, r0, col0);
                    const int kr0 = r0 - (item_at(it) % p.chunks) * p.chunk;  // the sequence's row 0
                    const int nblk = (cnt + 127) / 128;
                    for (int j = 0; j < nblk; ++j, ++gb) {
                        const int s = gb & 1;
                        if (gb >= 2) mbar_wait(bar_ke + s, ((gb >> 1) - 1) & 1);
                        mbar_arrive_expect_tx(bar_kf + s, L::kKV);
                        for (int hf = 0; hf < L::kHalves; ++hf)
                            tma_load_2d(&tm_k, bar_kf + s, sk + s * L::kKV + hf * L::kStrip,
                                        col0 + hf * 64, kr0 + j * 128);
                        if (gb >= 2) mbar_wait(bar_ve + s, ((gb >> 1) - 1) & 1);
                        mbar_arrive_expect_tx(bar_vf + s, L::kKV);
                        for (int hf = 0; hf < L::kHalves; ++hf)
                            tma_load_2d(&tm_v, bar_vf + s, sv + s * L::kKV + hf * L::kStrip,
                                        col0 + hf * 64, kr0 + j * 128);
                    }
                }
            }
        } else if (warp == 3) {
            if (lane == 0 && p.stage_base) {
                // ---------------------------------------------------- staged base / out I/O
                const int nbox = (p.chunk + 63) >> 6;
                auto issue_base = [&](int it) {
                    int r0, col0;
                    item_rows(it, r0, col0);
                    fence_proxy_async_smem();  // prior generic reads of X before the refill
                    mbar_arrive_expect_tx(bar_bf, (uint32_t)(L::kHalves * nbox) * 8192u);
                    for (int hf = 0; hf < L::kHalves; ++hf)
                        for (int bx = 0; bx < nbox; ++bx)
                            tma_load_2d(&tm_b, bar_bf, sx + hf * p.x_strip + bx * 8192,
                                        col0 + hf * 64, r0 + bx * 64);
                };
                int cnt = 0;
                int it = next_live(blockIdx.x, cnt);
                if (it < items) issue_base(it);
                for (uint32_t li = 0; it < items; ++li) {
                    int r0, col0;
                    item_rows(it, r0, col0);
                    const int nx = next_live(it + gridDim.x, cnt);
                    mbar_wait(bar_xc, li & 1);
                    fence_proxy_async_smem();
                    for (int hf = 0; hf < L::kHalves; ++hf)
                        for (int bx = 0; bx < nbox; ++bx)
                            tma_store_2d(&tm_o, sx + hf * p.x_strip + bx * 8192, col0 + hf * 64,
                                         r0 + bx * 64);
                    bulk_commit();
                    bulk_wait_read0();  // X read out before it is refilled
                    if (nx < items) issue_base(nx);
                    it = nx;
                }
                bulk_wait0();
            }
        } else if (warp == 1) {
            // -------------------------------------------------------- MMA issuer
            // The whole warp walks the schedule (warp-uniform descriptors); the elected lane
            // issues every MMA and commit.
            constexpr uint32_t idS = idesc_bf16(128, 128, false, false);
            constexpr uint32_t idO = idesc_bf16(128, E, false, true);
            const uint32_t sK = smem_u32(sk), sV = smem_u32(sv);
            auto commit = [&](uint64_t* b) {
                if (elect_one()) mma_commit(b);
                __syncwarp();
            };
            auto issue_s = [&](int t, uint32_t g) {  // S_t = Q_t K_g^T
                const uint32_t qb = smem_u32(smem + p.off_q[t]);
                const uint32_t kb = sK + (g & 1) * L::kKV;
                uint64_t da[E / 16], db[E / 16];
#pragma unroll
                for (int kk = 0; kk < E / 16; ++kk) {
                    da[kk] = desc_kmajor_sw128(qb + (kk / 4) * p.q_strip[t] + (kk % 4) * 32);
                    db[kk] = desc_kmajor_sw128(kb + (kk / 4) * L::kStrip + (kk % 4) * 32);
                }
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < E / 16; ++kk)
                        mma_bf16(tmem + t * 128, da[kk], db[kk], idS, kk > 0 ? 1u : 0u);
                    mma_commit(bar_s + t);
                }
                __syncwarp();
            };
            auto issue_pv = [&](int t, uint32_t g, bool acc) {  // O_t (+)= P_t V_g
                const uint32_t vb = sV + (g & 1) * L::kKV;
                uint64_t dv[8];
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) dv[kk] = desc_mnmajor_sw128(vb + kk * 2048, L::kStrip);
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        mma_bf16_ts(tmem + L::kOcol + t * E, tmem + t * 128 + kk * 8, dv[kk], idO,
                                    (acc || kk > 0) ? 1u : 0u);
                }
                __syncwarp();
            };
            auto wait_k = [&](uint32_t g) {
                mbar_wait(bar_kf + (g & 1), (g >> 1) & 1);
                if (cpa) fence_proxy_async_smem();  // cp.async (generic proxy) -> tcgen05 reads
                tc_fence_after();
            };
            int cnt = 0;
            int it = next_live(blockIdx.x, cnt);
            if (it < items) {
                uint32_t li = 0, g = 0;
                int j = 0, nblk = (cnt + 127) / 128;
                // the next live item, looked up while this one runs (its count load is off
                // the item boundary's critical path)
                int nx_cnt = 0;
                int nx_it = next_live(it + gridDim.x, nx_cnt);
                // prologue: both tiles' first S
                mbar_wait(bar_q + 0, 0);
                wait_k(0);
                issue_s(0, 0);
                if (nblk == 1) commit(bar_qe + 0);
                mbar_wait(bar_q + 1, 0);
                tc_fence_after();
                issue_s(1, 0);
                commit(bar_ke + 0);
                if (nblk == 1) commit(bar_qe + 1);
                while (true) {
                    const bool last = j == nblk - 1;
                    int nit = it, ncnt = cnt, nnblk = nblk, nj = j + 1;
                    uint32_t nli = li;
                    if (last) {
                        nit = nx_it;
                        ncnt = nx_cnt;
                        nnblk = (ncnt + 127) / 128;
                        nj = 0;
                        nli = li + 1;
                    }
                    const bool has_next = nit < items;
                    const bool nlast = has_next && nj == nnblk - 1;
                    const uint32_t gn = g + 1;
                    // ---- tile 0: P_0 V_g, then S_0 of the next block (this item or the next)
                    mbar_wait(bar_p + 0, g & 1);
                    if (lane == 0) PP_TRACE(2, g);
                    mbar_wait(bar_vf + (g & 1), (g >> 1) & 1);
                    if (cpa) fence_proxy_async_smem();
                    tc_fence_after();
                    if (lane == 0) PP_TRACE(3, g);
                    issue_pv(0, g, j > 0);
                    if (last) commit(bar_o + 0);
                    if (has_next) {
                        if (last) mbar_wait(bar_q + 0, nli & 1);
                        if (lane == 0) PP_TRACE(4, gn);
                        wait_k(gn);
                        if (lane == 0) PP_TRACE(5, gn);
                        issue_s(0, gn);  // in order after P_0 V_g: P_0 consumed first
                        if (nlast) commit(bar_qe + 0);
                    }
                    // ---- tile 1
                    mbar_wait(bar_p + 1, g & 1);
                    tc_fence_after();
                    if (lane == 0) PP_TRACE(6, g);
                    issue_pv(1, g, j > 0);
                    commit(bar_ve + (g & 1));
                    if (last) commit(bar_o + 1);
                    if (has_next) {
                        if (last) {
                            mbar_wait(bar_q + 1, nli & 1);
                            tc_fence_after();
                        }
                        issue_s(1, gn);
                        commit(bar_ke + (gn & 1));
                        if (nlast) commit(bar_qe + 1);
                    }
                    if (!has_next) break;
                    g = gn;
                    if (last) {
                        it = nit;
                        cnt = ncnt;
                        nblk = nnblk;
                        li = nli;
                        j = 0;
                        nx_it = next_live(it + gridDim.x, nx_cnt);
                    } else {
                        ++j;
                    }
                }
            }
        } else if (cpa) {
            // -------------------------------------------------------- sparse K/V row copies
            // copy thread ct owns the fixed 16-byte pieces (row r0 + kRowStep i, column piece
            // c16) of every block, written straight into the 128B-swizzled strips; rows past
            // the chunk's count are zero-filled (src-size 0), so dead key columns hold zeros.
            const int ct = cp_thread;
            const int c16 = ct % (E / 8), r0 = ct / (E / 8);
            const uint32_t cbase = (uint32_t)(c16 >> 3) * L::kStrip;
            const int64_t rs = p.layout == CSD_LAYOUT_BHNE ? E : (int64_t)p.heads * E;
            const uint32_t sK = smem_u32(sk), sV = smem_u32(sv);
            // indices one block ahead (the next block's loads are in flight while this
            // block's V rows are issued and the next K slot is awaited); the first block's
            // indices and the next item's count were loaded before the setup barrier
            int it = cp_it, cnt = cp_cnt, j = 0;
            int nx_cnt = 0;
            int nx_it = it < items ? next_live(it + gridDim.x, nx_cnt) : items;
            int32_t id[kCpRows];
#pragma unroll
            for (int i = 0; i < kCpRows; ++i) id[i] = cp_id[i];
            for (uint32_t g = 0; it < items; ++g) {
                const int bh = item_at(it) / p.chunks;
                const int64_t o0 = pp_tok_off(p.layout, bh / p.heads, bh % p.heads, 0, p.heads, p.n, E) + c16 * 8;
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
                if (ct == 0) PP_TRACE(0, g);
#pragma unroll
                for (int i = 0; i < kCpRows; ++i) {
                    const uint32_t row = (uint32_t)(r0 + kRowStep * i);
                    if (row < 128u)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                                         sK + s * L::kKV + cbase + sw128_offset(row, (uint32_t)(c16 & 7))),
                                     "l"(kb + (id[i] >= 0 ? (int64_t)id[i] * rs : 0)),
                                     "r"(id[i] >= 0 ? 16u : 0u)
                                     : "memory");
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                                 smem_u32(bar_kf + s))
                             : "memory");
                int32_t idn[kCpRows];
                load_ids(nit, ncnt, nj, idn);
                if (nj == 0 && nit < items) nx_it = next_live(nit + gridDim.x, nx_cnt);
                if (g >= 2) mbar_wait(bar_ve + s, ((g >> 1) - 1) & 1);
                if (ct == 0) PP_TRACE(1, g);
#pragma unroll
                for (int i = 0; i < kCpRows; ++i) {
                    const uint32_t row = (uint32_t)(r0 + kRowStep * i);
                    if (row < 128u)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                                         sV + s * L::kKV + cbase + sw128_offset(row, (uint32_t)(c16 & 7))),
                                     "l"(vb + (id[i] >= 0 ? (int64_t)id[i] * rs : 0)),
                                     "r"(id[i] >= 0 ? 16u : 0u)
                                     : "memory");
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                                 smem_u32(bar_vf + s))
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
        const int rows_t = p.rows[t];
        const int row = quad * 32 + lane;  // TMEM lane = row of tile t
        const int crow = t * 128 + row;    // row within the item
        const bool row_ok = row < rows_t;
        // Code warm-up (p.warm): before its first real item a softmax warp runs one DRY item
        // through the same code -- two key blocks (a full and a partial one) and the
        // epilogue -- with every barrier wait / arrive and every memory store switched off
        // and its P stores aimed at O (rewritten by the first P V, which waits for this
        // warp's real bar_p arrive).  The first pass through the unrolled softmax and
        // epilogue otherwise costs ~15k cycles of instruction fetches on every CTA's
        // critical path (worse after a GEMM evicted the code from L2).  warm 1: only the
        // warps holding no live row (tile 1 of a 192-row chunk) run it, concurrently with
        // the live warps' wait for their first S; warm 2: every softmax warp does.
        const bool live = quad * 32 < rows_t;
        bool dry = p.warm >= 2 || (p.warm == 1 && !live);
        if (live || dry) {
            const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
            const uint32_t tS = tmem + lane_off + t * 128;
            const uint32_t tO = tmem + lane_off + L::kOcol + t * E;
            const float sl2 = p.qk_scale_log2;
            const bool has_base = p.base != nullptr;
            uint32_t g = 0, li = 0;
            int cnt_nx = 0;
            bool waited = false;  // the dry pass reads no global memory: it runs before pdl_wait
            for (int it = blockIdx.x; it < items;) {
                if (!dry && !waited) {
                    pdl_wait();
                    waited = true;
                    cnt_nx = count_of(it);
                }
                const int cnt = dry ? 128 + 67 : cnt_nx;  // next count loaded one item ahead
                if (!dry && it + (int)gridDim.x < items) cnt_nx = count_of(it + gridDim.x);
                const int item = dry ? it : item_at(it);
                const int c = item % p.chunks, bh = item / p.chunks;
                const int b = bh / p.heads, h = bh % p.heads;
                const int64_t tok = (int64_t)c * p.chunk + crow;
                if (cnt == 0) {  // pass base through (attention.cpp:169)
                    if (row_ok && has_base && p.base != p.out) {
                        const int64_t off = pp_tok_off(p.layout, b, h, tok, p.heads, p.n, E);
                        const uint4* src = reinterpret_cast<const uint4*>(p.base + off);
                        uint4* dst = reinterpret_cast<uint4*>(p.out + off);
#pragma unroll
                        for (int q = 0; q < E / 8; ++q) dst[q] = src[q];
                    }
                    it += gridDim.x;
                    continue;
                }
                const bool wait = live && !dry;
                if (threadIdx.x == 128 * (t + 1)) PP_TRACE(22 + t, li);  // item set up
                const uint32_t tP = dry ? tO : tS;  // P destination
                const int nblk = (cnt + 127) / 128;
                float m_run = -INFINITY, m_true = -INFINITY, l_run = 0.f;
                for (int j = 0; j < nblk; ++j) {
                    const int ncols = min(128, cnt - j * 128);
                    if (wait) mbar_wait(bar_s + t, g & 1);
                    tc_fence_after();
                    if (threadIdx.x == 128 * (t + 1)) PP_TRACE(7 + 2 * t, g);
                    uint32_t sr[128];
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        tmem_ld32(tS + q * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[q * 32]));
                    tmem_ld_wait();
                    if (threadIdx.x == 128 * (t + 1)) PP_TRACE(16 + t, g);
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
                            mx4[u] = fmax3(mx4[u], __uint_as_float(sr[i + 2 * u]),
                                           __uint_as_float(sr[i + 2 * u + 1]));
                    const float mraw = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
                    const float mx = row_ok ? mraw * sl2 : -INFINITY;  // sl2 > 0: max commutes
                    m_true = fmaxf(m_true, mx);
                    const bool need = mx > m_run + kRescaleThreshold;
                    const float alpha = need ? ex2_approx(m_run - mx) : 1.0f;
                    if (need) {
                        m_run = mx;
                        l_run *= alpha;
                    }
                    if (threadIdx.x == 128 * (t + 1)) PP_TRACE(18 + t, g);
                    const float neg_m = row_ok ? -m_run : -INFINITY;  // dead rows -> p = 0
                    const float2 sl2v = make_float2(sl2, sl2), nm2 = make_float2(neg_m, neg_m);
                    float2 part0 = make_float2(0.f, 0.f), part1 = make_float2(0.f, 0.f);
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        uint32_t pk[16];
                        if (cc * 32 >= ncols) {  // uniform: a fully masked group, P = 0
#pragma unroll
                            for (int q = 0; q < 16; ++q) pk[q] = 0u;
                        } else {
                            // 2^(S*scale - m) with paired FFMA2 / FADD2 (two sums in flight)
#pragma unroll
                            for (int q = 0; q < 16; ++q) {
                                const float2 x = make_float2(__uint_as_float(sr[cc * 32 + 2 * q]),
                                                             __uint_as_float(sr[cc * 32 + 2 * q + 1]));
                                const float2 y = __ffma2_rn(x, sl2v, nm2);
                                float2 e;
                                if (kPoly > 0 && (q % (kPoly > 0 ? kPoly : 1)) == kPoly - 1) {
                                    e = ex2_poly2(y);  // FMA pipe: relieves MUFU (FA4's split)
                                } else {
                                    e.x = ex2_approx(y.x);
                                    e.y = ex2_approx(y.y);
                                }
                                if (q & 1) part1 = __fadd2_rn(part1, e);
                                else part0 = __fadd2_rn(part0, e);
                                pk[q] = pack_bf16x2(e.x, e.y);
                            }
                        }
                        // P_t (bf16 pairs) over S_t columns [16 cc, 16 cc + 16): every S
                        // column of this block is already in registers
                        tmem_st16(tP + cc * 16, pk);
                    }
                    const float2 part = __fadd2_rn(part0, part1);
                    l_run += part.x + part.y;
                    if (threadIdx.x == 128 * (t + 1)) PP_TRACE(20 + t, g);
                    // O_t holds P V of the earlier blocks (complete: S_t(g) was issued after
                    // P_t V_{g-1}); rescale it before this block's P V accumulates (after the
                    // P stores, when the S row no longer occupies registers)
                    if (j > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll 1
                        for (int oc = 0; oc < E / 32; ++oc) {
                            uint32_t r[32];
                            tmem_ld32(tO + oc * 32, r);
                            tmem_ld_wait();
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                            tmem_st32(tO + oc * 32, r);
                        }
                    }
                    tmem_st_wait();
                    tc_fence_before();
                    if (threadIdx.x == 128 * (t + 1)) PP_TRACE(8 + 2 * t, g);
                    if (wait) {
                        mbar_arrive(bar_p + t);
                        ++g;
                    }
                }
                // -------------------------------------------------------- epilogue
                if (wait) mbar_wait(bar_o + t, li & 1);
                tc_fence_after();
                if (threadIdx.x == 128 * (t + 1)) PP_TRACE(11 + t, 2 * li);
                if (p.stage_base) {
                    // out = base + scale * O / l with the item's base tile in smem (TMA,
                    // issued after the previous item's out store); rows combined in place,
                    // the I/O thread stores the tile by TMA
                    if (wait) mbar_wait(bar_bf, li & 1);
                    const float fsc = p.scale / l_run;
                    uint32_t ro[E];
#pragma unroll
                    for (int oc = 0; oc < E / 32; ++oc)
                        tmem_ld32(tO + oc * 32, *reinterpret_cast<uint32_t(*)[32]>(&ro[oc * 32]));
                    tmem_ld_wait();
                    // per 64-column strip: the row's 8 base pieces loaded together, then
                    // combined and stored (independent loads in flight, not a load-use chain)
#pragma unroll
                    for (int hf = 0; hf < E / 64; ++hf) {
                        if (!row_ok) continue;
                        uint8_t* rowp = sx + hf * p.x_strip + crow * 128;
                        uint4 bv[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            bv[q] = *reinterpret_cast<const uint4*>(rowp + ((q ^ (crow & 7)) << 4));
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&bv[q]);
                            const uint32_t* r = ro + hf * 64 + q * 8;
                            uint32_t o4[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const float2 f = __bfloat1622float2(b2[u]);
                                o4[u] = pack_bf16x2(fmaf(fsc, __uint_as_float(r[2 * u]), f.x),
                                                    fmaf(fsc, __uint_as_float(r[2 * u + 1]), f.y));
                            }
                            st_shared_v4_if(!dry, rowp + ((q ^ (crow & 7)) << 4), o4);  // dry pass: no store
                        }
                    }
                    fence_proxy_async_smem();  // in-place writes -> async proxy (TMA store)
                    __syncwarp();
                    if (lane == 0 && wait) mbar_arrive(bar_xc);
                } else {
                    const int64_t off = pp_tok_off(p.layout, b, h, tok, p.heads, p.n, E);
                    const float inv_l = 1.0f / l_run;
                    uint32_t ro[E];
#pragma unroll
                    for (int oc = 0; oc < E / 32; ++oc)
                        tmem_ld32(tO + oc * 32, *reinterpret_cast<uint32_t(*)[32]>(&ro[oc * 32]));
                    tmem_ld_wait();
#pragma unroll
                    for (int oc = 0; oc < E / 32; ++oc) {
                        const uint32_t* r = ro + oc * 32;
                        if (!row_ok) continue;
                        uint4 bq[4];
                        if (has_base) {
                            const uint4* bp = reinterpret_cast<const uint4*>(p.base + off + oc * 32);
#pragma unroll
                            for (int q = 0; q < 4; ++q) bq[q] = __ldg(bp + q);
                        }
                        uint4* dp = reinterpret_cast<uint4*>(p.out + off + oc * 32);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            float o[8];
#pragma unroll
                            for (int i = 0; i < 8; ++i) o[i] = __uint_as_float(r[q * 8 + i]) * inv_l;
                            if (has_base) {
                                const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&bq[q]);
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    const float2 f = __bfloat1622float2(b2[u]);
                                    o[2 * u] = f.x + p.scale * o[2 * u];
                                    o[2 * u + 1] = f.y + p.scale * o[2 * u + 1];
                                }
                            }
                            uint4 v;
                            v.x = pack_bf16x2(o[0], o[1]);
                            v.y = pack_bf16x2(o[2], o[3]);
                            v.z = pack_bf16x2(o[4], o[5]);
                            v.w = pack_bf16x2(o[6], o[7]);
                            st_global_v4_if(!dry, dp + q, v);
                        }
                    }
                }
                if (row_ok && !dry && p.row_max != nullptr) {
                    const int64_t si = (int64_t)bh * p.n + tok;
                    p.row_max[si] = m_true * kLn2;
                    p.exp_sum[si] = l_run * exp2f(m_run - m_true);
                }
                tc_fence_before();  // O reads ordered before the next item's bar_p arrive
                if (threadIdx.x == 128 * (t + 1)) PP_TRACE(11 + t, 2 * li + 1);
                if (dry) {  // the real items follow (a warp without live rows is done)
                    dry = false;
                    if (!live) break;
                    continue;
                }
                ++li;
                it += gridDim.x;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0 && p.span != nullptr) p.span[2 * blockIdx.x + 1] = pp_globaltimer();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<L::kTmemCols>(tmem);
    }
}

uint64_t* h_pp_span = nullptr;
uint64_t* h_pp_trace = nullptr;

template <int E>
cudaError_t launch_pp(const AttnTcArgs& a, cudaStream_t s) {
    using L = PPLayout<E>;
    const uint64_t cols = a.layout == CSD_LAYOUT_BHNE ? E : (uint64_t)a.heads * E;
    const uint64_t rows = a.layout == CSD_LAYOUT_BHNE ? (uint64_t)(a.batch * a.heads * a.n)
                                                      : (uint64_t)(a.batch * a.n);
    CUtensorMap tq, tk, tv, tb, to;
    if (!make_map_bf16(&tq, a.q, cols, rows, cols, 64) ||
        !make_map_bf16(&to, a.out, cols, rows, cols, 64) ||
        !make_map_bf16(&tb, a.base != nullptr ? a.base : a.q, cols, rows, cols, 64) ||
        !make_map_bf16(&tk, a.k, cols, rows, cols, 128) ||
        !make_map_bf16(&tv, a.v, cols, rows, cols, 128))
        return cudaErrorInvalidValue;
    PPParams p{};
    p.idx = a.idx;
    p.counts = a.counts;
    p.k_max = a.k_max;
    p.base = static_cast<const __nv_bfloat16*>(a.base);
    p.out = static_cast<__nv_bfloat16*>(a.out);
    p.scale = a.scale;
    p.row_max = a.row_max;
    p.exp_sum = a.exp_sum;
    p.layout = a.layout;
    p.heads = (int)a.heads;
    p.n = (int)a.n;
    p.chunk = (int)a.chunk;
    p.chunks = (int)(a.n / a.chunk);
    p.items = (int)(a.batch * a.heads * p.chunks);
    p.kp = static_cast<const __nv_bfloat16*>(a.k);
    p.vp = static_cast<const __nv_bfloat16*>(a.v);
    p.qk_scale_log2 = kLog2e / std::sqrt((float)E);
    p.span = h_pp_span;
    p.order = a.order;
    {
        static const int warm = [] {
            const char* e = std::getenv("CSD_PP_WARM");
            return e ? std::atoi(e) : 1;
        }();
        p.warm = warm;
    }
    p.trace = h_pp_trace;
    auto al = [](uint32_t v) { return (v + 1023u) & ~1023u; };
    uint32_t off = 0;
    for (int t = 0; t < 2; ++t) {
        p.rows[t] = (int)std::min<int64_t>(128, a.chunk - 128 * t);
        p.q_rows[t] = (p.rows[t] + 63) / 64 * 64;
        p.off_q[t] = off;
        p.q_strip[t] = (uint32_t)p.q_rows[t] * 128u;
        off = al(off + L::kHalves * p.q_strip[t]);
    }
    const uint32_t xrows = (uint32_t)((a.chunk + 63) / 64 * 64);
    const uint32_t xbytes = L::kHalves * xrows * 128u;
    const uint32_t tail = 4 * L::kKV + 256;
    p.stage_base = (a.base != nullptr && off + xbytes + tail <= L::kMaxSmem) ? 1 : 0;
    p.x_strip = xrows * 128u;
    p.off_x = off;
    if (p.stage_base) off = al(off + xbytes);
    p.off_k = off;
    p.off_v = off + 2 * L::kKV;
    p.off_bar = p.off_v + 2 * L::kKV;
    const uint32_t smem_bytes = p.off_bar + 256;
    if (smem_bytes > L::kMaxSmem) return cudaErrorNotSupported;
    // exponential split: dense passes (MUFU-bound, 36 blocks per item) put every 4th pair on
    // the FMA pipe (FLUX dense 254 -> 240 us); sparse items (3 blocks, latency-bound) measured
    // slower with it (53 -> 57 us).  CSD_PP_POLY overrides.
    static const int poly_env = [] {
        const char* e = std::getenv("CSD_PP_POLY");
        return e ? std::atoi(e) : -1;
    }();
    const int poly = poly_env >= 0 ? poly_env : (a.idx == nullptr ? 4 : 0);
    // dense passes: poly 4 by default, no LPT order; sparse items: poly 0, LPT order optional
    auto kern = a.idx == nullptr ? (poly == 4 ? k_attn_pp<E, 4, false, true> : k_attn_pp<E, 0, false, true>)
                : a.order != nullptr ? (poly == 4 ? k_attn_pp<E, 4, true, false> : k_attn_pp<E, 0, true, false>)
                                     : (poly == 4 ? k_attn_pp<E, 4, false, false> : k_attn_pp<E, 0, false, false>);
    cudaError_t err = ensure_smem_attr(kern, (int)L::kMaxSmem);
    if (err != cudaSuccess) return err;
    const unsigned grid = (unsigned)std::min<int64_t>(p.items, sm_count());
    return launch_ex_pdl(1, kern, dim3(grid), dim3(L::kThreads), smem_bytes, s, 1, tq, tk, tv, tb, to, p);
}

}  // namespace

namespace {
// Stable counting sort of the items by descending key-block count (ties keep item order, so
// uniform counts give the identity -- the strided order whose concurrent items share heads
// in L2).  order[items] = 1 flags the identity, letting the attention kernel skip the
// indirection.  Tiles of 1024 items: per-warp bin counts, a cross-warp scan per bin, ranks
// within a warp by __match_any_sync.
constexpr int kLptBins = 64;  // key-block counts >= 63 share the first bin
__global__ void __launch_bounds__(1024) k_lpt_order(const int32_t* __restrict__ counts, int items,
                                                    int block_keys, int32_t* __restrict__ order) {
    __shared__ int hist[kLptBins], base[kLptBins];
    __shared__ int wcnt[32][kLptBins];
    __shared__ int not_ident;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kLptBins; i += blockDim.x) hist[i] = 0;
    if (threadIdx.x == 0) not_ident = 0;
    __syncthreads();
    auto bin_of = [&](int it) {
        const int nb = (max(counts[it], 0) + block_keys - 1) / block_keys;
        return kLptBins - 1 - min(nb, kLptBins - 1);  // more blocks -> earlier bin
    };
    for (int it = threadIdx.x; it - lane < items; it += blockDim.x) {
        const int b = it < items ? bin_of(it) : -1;
        const unsigned m = __match_any_sync(0xffffffffu, b);
        if (lane == __ffs(m) - 1 && b >= 0) atomicAdd(&hist[b], __popc(m));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0, used = 0;
        for (int b = 0; b < kLptBins; ++b) {
            base[b] = run;
            run += hist[b];
            used += hist[b] > 0;
        }
        if (used > 1) not_ident = 1;  // one bin only: the stable order is the identity
    }
    __syncthreads();
    for (int t0 = 0; t0 < items; t0 += blockDim.x) {
        const int it = t0 + threadIdx.x;
        const int b = it < items ? bin_of(it) : -1;
        const unsigned m = __match_any_sync(0xffffffffu, b);
        const int rank = __popc(m & ((1u << lane) - 1u));
        for (int i = threadIdx.x; i < 32 * kLptBins; i += blockDim.x) (&wcnt[0][0])[i] = 0;
        __syncthreads();
        if (b >= 0 && lane == __ffs(m) - 1) wcnt[warp][b] = __popc(m);
        __syncthreads();
        if (threadIdx.x < kLptBins) {  // exclusive scan over warps, per bin
            int run = base[threadIdx.x];
            for (int w = 0; w < 32; ++w) {
                const int c = wcnt[w][threadIdx.x];
                wcnt[w][threadIdx.x] = run;
                run += c;
            }
            base[threadIdx.x] = run;
        }
        __syncthreads();
        if (b >= 0) order[wcnt[warp][b] + rank] = it;
        __syncthreads();
    }
    if (threadIdx.x == 0) order[items] = not_ident ? 0 : 1;
}
}  // namespace

cudaError_t lpt_order(const int32_t* counts, int64_t items, int64_t block_keys, int32_t* order,
                      cudaStream_t s) {
    k_lpt_order<<<1, 1024, 0, s>>>(counts, (int)items, (int)block_keys, order);
    return cudaGetLastError();
}

bool attn_pp_supported(const AttnTcArgs& a) {
    static const bool off = [] {
        const char* e = std::getenv("CSD_ATTN_KERNEL");
        return e != nullptr && std::string(e) == "tc";
    }();
    return !off && (a.e == 64 || a.e == 128) && a.colsum == nullptr && a.chunk > 128 &&
           a.chunk <= 256;
}

cudaError_t attn_pp(const AttnTcArgs& a, cudaStream_t s) {
    if (a.n % a.chunk) return cudaErrorInvalidValue;
    return a.e == 128 ? launch_pp<128>(a, s) : launch_pp<64>(a, s);
}

}  // namespace dev
}  // namespace csd

// Debug only: per-CTA [start, end] globaltimer stamps of the ping-pong kernel (2 x grid).
extern "C" int csd_debug_set_attn_pp_span(void* dev_buf) {
    csd::dev::h_pp_span = static_cast<uint64_t*>(dev_buf);
    return 0;
}
// Debug only: clock64 timeline of the first kPPTraceCtas CTAs (8 x 2048 uint64; null: off).
extern "C" int csd_debug_set_attn_pp_trace(void* dev_buf) {
    csd::dev::h_pp_trace = static_cast<uint64_t*>(dev_buf);
    return 0;
}
