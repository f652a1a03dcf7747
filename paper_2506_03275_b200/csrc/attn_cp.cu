// attn_cp.cu — column-sparse delta attention on CTA PAIRS (cta_group::2), CSD_MODE_PROD.
//
// Replaces sparse_delta_attention (attention.cpp:147-194) for query chunks of 192 / 256 rows
// (FLUX and Hunyuan chunk 192): out = base + scale * softmax(Q_c K_S^T / sqrt(E)) V_S per
// (b, h, chunk c) with S the chunk's selected key set.
//
// Work item = one chunk, spread over a CLUSTER OF TWO SMs: the pair's M = 256 MMA tile holds
// the chunk's rows, R = chunk / 2 in each CTA (TMEM lanes 0..R-1; a 192-row chunk leaves 32
// dead lanes per CTA instead of a 64-live-row second tile on one SM).  Each CTA stages HALF
// of every key block: K rows of 64 of the block's 128 keys (the S MMA's B operand is split by
// N) and the 128 keys' V rows restricted to 64 of the E columns (the P V MMA's B is split by
// N = E).  So per SM the gather bytes of a block halve, and the tensor core of both SMs works
// on every MMA the leader issues.
//
// TMEM (512 columns per CTA): S double buffer [0,128) / [128,256) (P aliased over the first
// 64 columns of its S as bf16 pairs, TS-form P V), O double buffer [256,384) / [384,512).
// The MMA issuer keeps S two key blocks ahead of P V (S(g+2) is issued right after P V(g)),
// so the softmax of block g+1 never waits for P V(g), and the O buffers alternate per item
// so one item's epilogue overlaps the next item's P V.
//
// Roles per CTA (16 warps): warp 0 lane 0 Q loader (TMA, this CTA's R rows; bytes on the
// leader's barrier), lane 1 gather relay (local cp.async completion -> the leader's
// barrier), lane 31 staged base / out I/O; warp 1 MMA issuer (leader CTA only); warps 2-3,
// 12-15 K/V row gathers (cp.async, 16-byte pieces into 128B-swizzled strips, rows past the
// chunk's count zero-filled); warps 4-11 softmax + epilogue, TWO warps per TMEM lane quadrant
// (64 key columns each; the row maxima and sums are exchanged through shared memory).
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

uint64_t* h_cp_trace = nullptr;

namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale O only when the max grows > 2^8
constexpr int E = 128;
constexpr uint32_t kThreads = 512;
constexpr uint32_t kQBuf = 2 * 128 * 128;     // one Q buffer: 2 strips x 128 rows x 128 B
constexpr uint32_t kKHalf = 2 * 64 * 128;     // 64 keys x 256 B (2 strips of 64 rows)
constexpr uint32_t kVHalf = 128 * 128;        // 128 keys x 64 E columns (MN-major)
constexpr uint32_t kMaxSmem = 227 * 1024;
constexpr int kMaxStages = 4;
constexpr int kCT = 128;  // K / V gather threads (warps 12-15)

struct CPParams {
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
    int rows;  // R: query rows per CTA (chunk / 2, multiple of 32)
    int ns;    // K/V ring stages
    uint32_t off_k, off_v, off_x, x_strip, off_bar;
    const int32_t* order;  // LPT item order or null
    uint64_t* trace;       // debug timeline (null: off): kCPTraceCtas x 2048 clock64 stamps
};

// Debug timeline (scripts/attn_cp_trace.py): CTAs < kCPTraceCtas stamp clock64() at slot
// event * 64 + (index & 63).
constexpr int kCPTraceCtas = 4;
#ifdef CSD_CP_NOTRACE
#define CP_TRACE(ev, ix) \
    do {                 \
    } while (0)
#else
#define CP_TRACE(ev, ix)                                                                     \
    do {                                                                                     \
        if (p.trace != nullptr && blockIdx.x < kCPTraceCtas)                                 \
            p.trace[blockIdx.x * 2048 + (ev) * 64 + ((ix) & 63)] = clock64();                \
    } while (0)
#endif

__device__ __forceinline__ int64_t cp_tok_off(int layout, int64_t b, int64_t h, int64_t tok, int heads,
                                              int n) {
    return layout == CSD_LAYOUT_BHNE ? (((b * heads + h) * (int64_t)n) + tok) * E
                                     : ((b * (int64_t)n + tok) * heads + h) * E;
}

// kPoly > 0: every kPoly-th exponential pair of a row runs as a degree-3 polynomial on the
// FMA pipe instead of MUFU (ex2_poly2), relieving the MUFU-bound softmax.
template <int kPoly>
__global__ void __launch_bounds__(kThreads, 1)
k_attn_cp(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_b,
          const __grid_constant__ CUtensorMap tm_o, const CPParams p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_u32 = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int items = p.items, R = p.rows, NS = p.ns;
    const int lw = 2 * (R >> 5);  // live softmax warps per CTA (two per lane quadrant)
    if (threadIdx.x == 0) CP_TRACE(31, 0);

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
    uint64_t* bar_q = bars + 0;     // [2] leader: Q buffer landed (both CTAs' bytes)
    uint64_t* bar_qe = bars + 2;    // [2] Q buffer free (the item's last S completed)
    uint64_t* kf_loc = bars + 4;    // [4] this CTA's K half of stage s landed (cp.async)
    uint64_t* vf_loc = bars + 8;    // [4]
    uint64_t* kf = bars + 12;       // [4] leader: both CTAs' K halves landed (relayed)
    uint64_t* vf = bars + 16;       // [4]
    uint64_t* kve = bars + 20;      // [4] stage s free (its P V completed)
    uint64_t* bar_s = bars + 24;    // [2] S buffer in TMEM
    uint64_t* bar_p = bars + 26;    // [2] leader: P in the S buffer (all live softmax warps)
    uint64_t* bar_pv = bars + 28;   // [2] P V of the buffer's block completed
    uint64_t* bar_o = bars + 30;    // [2] O buffer final for its item
    uint64_t* bar_oe = bars + 32;   // [2] leader: O buffer read out (all live softmax warps)
    uint64_t* bar_bf = bars + 34;   // staged base tile landed
    uint64_t* bar_xc = bars + 35;   // every live softmax warp combined its rows into X
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 36);
    uint8_t* const sq = smem;
    uint8_t* const sk = smem + p.off_k;
    uint8_t* const sv = smem + p.off_v;
    uint8_t* const sx = smem + p.off_x;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar_q + i, 1);
            mbar_init(bar_qe + i, 1);
            mbar_init(bar_s + i, 1);
            mbar_init(bar_p + i, 2u * lw);
            mbar_init(bar_pv + i, 1);
            mbar_init(bar_o + i, 1);
            mbar_init(bar_oe + i, 2u * lw);
        }
        for (int s = 0; s < kMaxStages; ++s) {
            mbar_init(kf_loc + s, kCT);
            mbar_init(vf_loc + s, kCT);
            mbar_init(kf + s, 2);
            mbar_init(vf + s, 2);
            mbar_init(kve + s, 1);
        }
        mbar_init(bar_bf, 1);
        mbar_init(bar_xc, (uint32_t)lw);

        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    if (threadIdx.x == 0) pdl_trigger();

    const int32_t* order = (p.order != nullptr && p.order[items] == 0) ? p.order : nullptr;
    auto item_at = [&](int pos) -> int { return order != nullptr ? order[pos] : pos; };
    auto count_of = [&](int pos) -> int { return p.counts[item_at(pos)]; };
    auto next_live = [&](int from, int& cnt_out) -> int {  // next live item position of this pair
        int x = from;
        cnt_out = 0;
        for (; x < items; x += npairs) {
            cnt_out = count_of(x);
            if (cnt_out > 0) break;
        }
        return x;
    };
    // this CTA's first token row and head column of the item at position pos
    auto item_rows = [&](int pos, int& row0, int& col0) {
        const int it = item_at(pos);
        const int bh = it / p.chunks;
        row0 = p.layout == CSD_LAYOUT_BHNE ? bh * p.n : (bh / p.heads) * p.n;
        col0 = p.layout == CSD_LAYOUT_BHNE ? 0 : (bh % p.heads) * E;
        row0 += (it % p.chunks) * p.chunk + (int)rank * R;
    };

    // (setmaxnreg and the code it funds must share a branch: ptxas budgets registers per
    // region, and a merged dispatch falls back to the 128-register launch bound -- spills)
    if (warp < 4 || warp >= 12) {
        regs_dec<72>();
        if (warp == 0) {
            if (lane == 0) {
                // ---------------------------------------------------- Q loader (double buffer)
                tma_prefetch_desc(&tm_q);
                int cnt = 0;
                uint32_t li = 0;
                for (int it = next_live(pair, cnt); it < items; ++li) {
                    const uint32_t qb = li & 1;
                    if (li >= 2) mbar_wait(bar_qe + qb, ((li >> 1) - 1) & 1);
                    CP_TRACE(12, li);
                    if (rank == 0) mbar_arrive_expect_tx(bar_q + qb, 2u * (uint32_t)R * 256u);
                    int r0, col0;
                    item_rows(it, r0, col0);
                    for (int hf = 0; hf < 2; ++hf)
                        for (int bx = 0; bx < R / 32; ++bx)
                            tma_load_2d_pair(&tm_q, bar_q + qb, sq + qb * kQBuf + hf * 16384 + bx * 4096,
                                             col0 + hf * 64, r0 + bx * 32);
                    const int nx = next_live(it + npairs, cnt);
                    if (nx < items) {  // the next item's Q into L2 while this one runs
                        int nr0, ncol0;
                        item_rows(nx, nr0, ncol0);
                        for (int hf = 0; hf < 2; ++hf)
                            for (int bx = 0; bx < R / 32; ++bx)
                                tma_prefetch_2d(&tm_q, ncol0 + hf * 64, nr0 + bx * 32);
                    }
                    it = nx;
                }
            }
        } else if (warp == 2) {
            if (lane == 0) {
                // ---------------------------------------------------- gather relay
                // this CTA's cp.async completions (local barriers) -> the leader's barriers
                int cnt = 0;
                uint32_t g = 0;
                for (int it = next_live(pair, cnt); it < items; it = next_live(it + npairs, cnt)) {
                    const int nblk = (cnt + 127) >> 7;
                    for (int j = 0; j < nblk; ++j, ++g) {
                        const uint32_t s = g % NS, ph = (g / NS) & 1;
                        mbar_wait(kf_loc + s, ph);
                        CP_TRACE(2, g);
                        fence_proxy_async_smem();  // cp.async (generic proxy) -> tcgen05 reads
                        mbar_arrive_cluster(kf + s, 0);
                        mbar_wait(vf_loc + s, ph);
                        CP_TRACE(3, g);
                        fence_proxy_async_smem();
                        mbar_arrive_cluster(vf + s, 0);
                    }
                }
            }
        } else if (warp == 3) {
            if (lane == 0) {
                // ---------------------------------------------------- staged base / out I/O
                tma_prefetch_desc(&tm_b);
                tma_prefetch_desc(&tm_o);
                auto issue_base = [&](int it) {
                    int r0, col0;
                    item_rows(it, r0, col0);
                    fence_proxy_async_smem();  // prior generic reads of X before the refill
                    mbar_arrive_expect_tx(bar_bf, (uint32_t)R * 256u);
                    for (int hf = 0; hf < 2; ++hf)
                        for (int bx = 0; bx < R / 32; ++bx)
                            tma_load_2d(&tm_b, bar_bf, sx + hf * p.x_strip + bx * 4096, col0 + hf * 64,
                                        r0 + bx * 32);
                };
                auto prefetch_base = [&](int it) {
                    int r0, col0;
                    item_rows(it, r0, col0);
                    for (int hf = 0; hf < 2; ++hf)
                        for (int bx = 0; bx < R / 32; ++bx) tma_prefetch_2d(&tm_b, col0 + hf * 64, r0 + bx * 32);
                };
                int cnt = 0;
                int it = next_live(pair, cnt);
                if (it < items) issue_base(it);
                for (uint32_t li = 0; it < items; ++li) {
                    int r0, col0;
                    item_rows(it, r0, col0);
                    const int nx = next_live(it + npairs, cnt);
                    if (nx < items) prefetch_base(nx);
                    mbar_wait(bar_xc, li & 1);
                    fence_proxy_async_smem();
                    for (int hf = 0; hf < 2; ++hf)
                        for (int bx = 0; bx < R / 32; ++bx)
                            tma_store_2d(&tm_o, sx + hf * p.x_strip + bx * 4096, col0 + hf * 64, r0 + bx * 32);
                    bulk_commit();
                    bulk_wait_read0();  // X read out before it is refilled
                    if (nx < items) issue_base(nx);
                    it = nx;
                }
                bulk_wait0();
            }
        } else if (warp == 1) {
            if (rank == 0) {
                // ---------------------------------------------------- MMA issuer (leader)
                constexpr uint32_t idS = idesc_bf16(256, 128, false, false);
                constexpr uint32_t idO = idesc_bf16(256, E, false, true);
                const uint32_t sQ = smem_u32(sq), sK = smem_u32(sk), sV = smem_u32(sv);
                // two cursors over the pair's flattened key-block sequence: S runs two blocks
                // ahead of P V
                struct Cur {
                    int it, cnt, nblk, j;
                    uint32_t li, g;
                };
                auto start = [&](Cur& c) {
                    c.it = next_live(pair, c.cnt);
                    c.nblk = (c.cnt + 127) >> 7;
                    c.j = 0;
                    c.li = 0;
                    c.g = 0;
                };
                auto advance = [&](Cur& c) {
                    ++c.g;
                    if (++c.j == c.nblk) {
                        c.it = next_live(c.it + npairs, c.cnt);
                        c.nblk = (c.cnt + 127) >> 7;
                        c.j = 0;
                        ++c.li;
                    }
                };
                auto commit = [&](uint64_t* b) {
                    if (elect_one()) mma_commit_pair(b);
                    __syncwarp();
                };
                auto issue_s = [&](Cur& c) {
                    const uint32_t qb = c.li & 1, s = c.g % NS;
                    if (c.j == 0) mbar_wait(bar_q + qb, (c.li >> 1) & 1);
                    mbar_wait(kf + s, (c.g / NS) & 1);
                    fence_proxy_async_smem();
                    tc_fence_after();
                    if (lane == 0) CP_TRACE(4, c.g);
                    const uint32_t qa = sQ + qb * kQBuf, kb = sK + s * kKHalf;
                    uint64_t da[E / 16], db[E / 16];
#pragma unroll
                    for (int kk = 0; kk < E / 16; ++kk) {
                        da[kk] = desc_kmajor_sw128(qa + (kk / 4) * 16384 + (kk % 4) * 32);
                        db[kk] = desc_kmajor_sw128(kb + (kk / 4) * 8192 + (kk % 4) * 32);
                    }
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < E / 16; ++kk)
                            mma_bf16_pair(tmem + (c.g & 1) * 128, da[kk], db[kk], idS, kk > 0 ? 1u : 0u);
                        mma_commit_pair(bar_s + (c.g & 1));
                        if (c.j == c.nblk - 1) mma_commit_pair(bar_qe + qb);
                    }
                    __syncwarp();
                    advance(c);
                };
                Cur cs, cv;
                start(cs);
                start(cv);
                while (true) {
                    // S runs two blocks ahead of P V (one issue site: code size matters here)
                    while (cs.it < items && cs.g < cv.g + 2) issue_s(cs);
                    if (cv.it >= items) break;
                    const uint32_t g = cv.g, s = g % NS, ob = cv.li & 1;
                    mbar_wait(bar_p + (g & 1), (g >> 1) & 1);
                    if (lane == 0) CP_TRACE(5, g);
                    if (cv.j == 0 && cv.li >= 2) mbar_wait(bar_oe + ob, ((cv.li >> 1) - 1) & 1);
                    mbar_wait(vf + s, (g / NS) & 1);
                    fence_proxy_async_smem();
                    tc_fence_after();
                    if (lane == 0) CP_TRACE(6, g);
                    const uint32_t vb = sV + s * kVHalf;
                    uint64_t dv[8];
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) dv[kk] = desc_mnmajor_sw128(vb + kk * 2048, 8192);
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)
                            mma_bf16_ts_pair(tmem + 256 + ob * 128, tmem + (g & 1) * 128 + kk * 8, dv[kk], idO,
                                             (cv.j > 0 || kk > 0) ? 1u : 0u);
                        mma_commit_pair(kve + s);
                        mma_commit_pair(bar_pv + (g & 1));
                        if (cv.j == cv.nblk - 1) mma_commit_pair(bar_o + ob);
                    }
                    __syncwarp();
                    advance(cv);
                }
            }
        } else if (warp >= 12) {
            // -------------------------------------------------------- K / V row gathers
            // K: this CTA's 64 keys of every block (keys 64 rank .. +63), 16 pieces per row;
            // V: all 128 keys, the E columns [64 rank, +64), 8 pieces per row.  A block's
            // key ids are loaded one block ahead (the next item's too), off the issue path.
            const int ct = (warp - 12) * 32 + lane;
            constexpr int kKP = kCT / 16, kVP = kCT / 8;  // K / V rows per pass
            constexpr int kKN = 64 / kKP, kVN = 128 / kVP;  // passes
            const int kc = ct & 15, kr0 = ct >> 4;
            const int vc = ct & 7, vr0 = ct >> 3;
            const uint32_t sK = smem_u32(sk), sV = smem_u32(sv);
            const int64_t rs = p.layout == CSD_LAYOUT_BHNE ? E : (int64_t)p.heads * E;
            auto load_ids = [&](int pos, int cnt, int j, int32_t (&kid)[kKN], int32_t (&vid)[kVN]) {
                const int32_t* ids = p.idx + (int64_t)(pos < items ? item_at(pos) : 0) * p.k_max;
#pragma unroll
                for (int i = 0; i < kKN; ++i) {
                    const int kkey = j * 128 + (int)rank * 64 + kr0 + kKP * i;
                    kid[i] = (pos < items && kkey < cnt) ? __ldg(ids + kkey) : -1;
                }
#pragma unroll
                for (int i = 0; i < kVN; ++i) {
                    const int vkey = j * 128 + vr0 + kVP * i;
                    vid[i] = (pos < items && vkey < cnt) ? __ldg(ids + vkey) : -1;
                }
            };
            int cnt = 0;
            int it = next_live(pair, cnt);
            int32_t kid[kKN], vid[kVN];
            load_ids(it, cnt, 0, kid, vid);
            uint32_t g = 0;
            int j = 0;
            while (it < items) {
                const int item = item_at(it);
                const int bh = item / p.chunks;
                const int64_t o0 = cp_tok_off(p.layout, bh / p.heads, bh % p.heads, 0, p.heads, p.n);
                const __nv_bfloat16* kb = p.kp + o0 + kc * 8;
                const __nv_bfloat16* vb = p.vp + o0 + (int)rank * 64 + vc * 8;
                const int nblk = (cnt + 127) >> 7;
                // the next block (this item's or the next live item's first)
                int nit = it, ncnt = cnt, nj = j + 1;
                if (nj == nblk) {
                    nit = next_live(it + npairs, ncnt);
                    nj = 0;
                }
                int32_t nkid[kKN], nvid[kVN];
                load_ids(nit, ncnt, nj, nkid, nvid);
                const uint32_t s = g % NS;
                if (g >= (uint32_t)NS) mbar_wait(kve + s, ((g / NS) - 1) & 1);
                if (ct == 0) CP_TRACE(0, g);
                const uint32_t kst = sK + s * kKHalf + (uint32_t)(kc >> 3) * 8192u;
#pragma unroll
                for (int i = 0; i < kKN; ++i)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                                     kst + sw128_offset((uint32_t)(kr0 + kKP * i), (uint32_t)(kc & 7))),
                                 "l"(kb + (kid[i] >= 0 ? (int64_t)kid[i] * rs : 0)),
                                 "r"(kid[i] >= 0 ? 16u : 0u)
                                 : "memory");
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(kf_loc + s))
                             : "memory");
                const uint32_t vst = sV + s * kVHalf;
#pragma unroll
                for (int i = 0; i < kVN; ++i)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                                     vst + sw128_offset((uint32_t)(vr0 + kVP * i), (uint32_t)vc)),
                                 "l"(vb + (vid[i] >= 0 ? (int64_t)vid[i] * rs : 0)),
                                 "r"(vid[i] >= 0 ? 16u : 0u)
                                 : "memory");
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(vf_loc + s))
                             : "memory");
                if (ct == 0) CP_TRACE(1, g);
#pragma unroll
                for (int i = 0; i < kKN; ++i) kid[i] = nkid[i];
#pragma unroll
                for (int i = 0; i < kVN; ++i) vid[i] = nvid[i];
                it = nit;
                cnt = ncnt;
                j = nj;
                ++g;
            }
        }
    } else {
        regs_inc<184>();
        // ------------------------------------------------------------ softmax + epilogue
        // Warp w owns the 16 TMEM lanes [32 quad + 16 hh, +16) (tcgen05 16x32bx2 shapes):
        // threads t and t + 16 share a row, t < 16 holding key columns [0, 64), t >= 16
        // [64, 128) -- the row maximum and sum are one shuffle away, no cross-warp exchange.
        // (Measured alternatives: one warp per quadrant with 128 columns per thread and
        // dedicated epilogue warps, 80 us; two warps per quadrant splitting the columns with
        // a shared-memory max exchange, 65 us.)
        const int quad = warp & 3, hh = (warp - 4) >> 2, ch = lane >> 4;
        const int wrow0 = quad * 32 + hh * 16;  // first TMEM lane (row) of this warp
        if (wrow0 < R) {
            const int xr = wrow0 + (lane & 15);  // row within this CTA's rows
            const uint32_t lane_off = (uint32_t)wrow0 << 16;
            const float sl2 = p.qk_scale_log2;
            // epilogue of item `le` (run after the NEXT item's first key block, so the wait
            // for the item's last P V is off the softmax warps' path): out = base + scale O / l
            // into the staged base tile X, stored by the I/O thread
            auto epilogue = [&](uint32_t le, float lh) {
                const float l_row = lh + __shfl_xor_sync(0xffffffffu, lh, 16);
                const uint32_t ob = le & 1;
                mbar_wait(bar_o + ob, (le >> 1) & 1);
                tc_fence_after();
                if (threadIdx.x == 128) CP_TRACE(10, le);
                uint32_t ro[64];
                const uint32_t tO = tmem + lane_off + 256 + ob * 128;
                tmem_ld32_16x2<64>(tO, *reinterpret_cast<uint32_t(*)[32]>(&ro[0]));
                tmem_ld32_16x2<64>(tO + 32, *reinterpret_cast<uint32_t(*)[32]>(&ro[32]));
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(bar_oe + ob, 0);
                mbar_wait(bar_bf, le & 1);
                const float fsc = p.scale / l_row;
                uint8_t* rowp = sx + ch * p.x_strip;
                uint4 bv[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    bv[q] = *reinterpret_cast<const uint4*>(rowp + sw128_offset((uint32_t)xr, (uint32_t)q));
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&bv[q]);
                    uint32_t o4[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float2 f = __bfloat1622float2(b2[u]);
                        o4[u] = pack_bf16x2(fmaf(fsc, __uint_as_float(ro[q * 8 + 2 * u]), f.x),
                                            fmaf(fsc, __uint_as_float(ro[q * 8 + 2 * u + 1]), f.y));
                    }
                    *reinterpret_cast<uint4*>(rowp + sw128_offset((uint32_t)xr, (uint32_t)q)) =
                        make_uint4(o4[0], o4[1], o4[2], o4[3]);
                }
                fence_proxy_async_smem();  // in-place writes -> async proxy (TMA store)
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_xc);
                if (threadIdx.x == 128) CP_TRACE(11, le);
            };
            int pend = -1;  // item whose epilogue is pending
            float pend_l = 0.f;
            uint32_t g = 0, li = 0;
            // one extra pass after the last item drains the pending epilogue (a single copy of
            // the epilogue code: instruction fetch is a measured limiter here)
            for (int it = pair;; it += npairs) {
                const bool drain = it >= items;
                const int cnt = drain ? 0 : count_of(it);
                const int item = drain ? 0 : item_at(it);
                if (!drain && cnt == 0) {  // no selected key: out = base (attention.cpp:169)
                    if (p.base != p.out) {
                        const int c = item % p.chunks, bh = item / p.chunks;
                        const int64_t tok = (int64_t)c * p.chunk + (int)rank * R + xr;
                        const int64_t off = cp_tok_off(p.layout, bh / p.heads, bh % p.heads, tok, p.heads, p.n) + ch * 64;
                        const uint4* src = reinterpret_cast<const uint4*>(p.base + off);
                        uint4* dst = reinterpret_cast<uint4*>(p.out + off);
#pragma unroll
                        for (int q = 0; q < 8; ++q) dst[q] = src[q];
                    }
                    continue;
                }
                const int nblk = drain ? 1 : (cnt + 127) >> 7;
                float m_run = -INFINITY, l_half = 0.f;
                for (int j = 0; j < nblk; ++j) {
                    if (!drain) {
                        const int bcols = min(128, cnt - j * 128);  // live key columns of the block
                        const int ncols = bcols - ch * 64;          // ... of my half
                        const uint32_t tS = tmem + lane_off + (g & 1) * 128;
                        mbar_wait(bar_s + (g & 1), (g >> 1) & 1);
                        tc_fence_after();
                        if (lane == 0) CP_TRACE(hh ? 18 : 7, g + 64 * quad);
                        uint32_t sr[64];
                        tmem_ld32_16x2<64>(tS, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
                        tmem_ld32_16x2<64>(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
                        tmem_ld_wait();
                        if (bcols < 128) {  // uniform: the item's last, partial key block
#pragma unroll
                            for (int i = 0; i < 64; ++i)
                                if (i >= ncols) sr[i] = __float_as_uint(-INFINITY);
                        }
                        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                        for (int i = 0; i < 64; i += 8)
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                mx4[u] = fmax3(mx4[u], __uint_as_float(sr[i + 2 * u]), __uint_as_float(sr[i + 2 * u + 1]));
                        float mh = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
                        mh = fmaxf(mh, __shfl_xor_sync(0xffffffffu, mh, 16));
                        const float mx = mh * sl2;  // sl2 > 0: max commutes
                        if (lane == 0) CP_TRACE(hh ? 19 : 8, g + 64 * quad);
                        const bool need = mx > m_run + kRescaleThreshold;
                        const float alpha = need ? ex2_approx(m_run - mx) : 1.0f;
                        if (need) {
                            m_run = mx;
                            l_half *= alpha;
                        }
                        const float2 sl2v = make_float2(sl2, sl2), nm2 = make_float2(-m_run, -m_run);
                        float2 part0 = make_float2(0.f, 0.f), part1 = make_float2(0.f, 0.f);
#pragma unroll
                        for (int cc = 0; cc < 2; ++cc) {
                            uint32_t pk[16];
                            if (cc * 32 >= bcols) {  // uniform: a group masked in both halves, P = 0
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
                            // P (bf16 pairs) of keys [64 ch + 32 cc, +32) over S columns
                            // [32 ch + 16 cc, +16) (this warp's S loads completed above)
                            tmem_st16_16x2<32>(tS + cc * 16, pk);
                        }
                        const float2 part = __fadd2_rn(part0, part1);
                        l_half += part.x + part.y;
                        if (j > 0 && __any_sync(0xffffffffu, need)) {
                            // O holds P V of the earlier blocks once P V(g-1) completed
                            mbar_wait(bar_pv + ((g - 1) & 1), ((g - 1) >> 1) & 1);
                            tc_fence_after();
                            const uint32_t tO = tmem + lane_off + 256 + (li & 1) * 128;
#pragma unroll 1
                            for (int oc = 0; oc < 2; ++oc) {
                                uint32_t r[32];
                                tmem_ld32_16x2<64>(tO + oc * 32, r);
                                tmem_ld_wait();
#pragma unroll
                                for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                                tmem_st32_16x2<64>(tO + oc * 32, r);
                            }
                        }
                        tmem_st_wait();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_remote(bar_p + (g & 1), 0);
                        if (lane == 0) CP_TRACE(hh ? 23 : 9, g + 64 * quad);
                        ++g;
                    }
                    if (j == 0 && pend >= 0) {
                        epilogue((uint32_t)pend, pend_l);
                        pend = -1;
                    }
                }
                if (drain) break;
                pend = (int)li;
                pend_l = l_half;
                ++li;
            }
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair<512>(tmem);
    }
}

}  // namespace

// Opt-in (CSD_ATTN_CP=1 or csd_debug_set_attn_cp(1)): measured at FLUX / 93 % the pair kernel
// takes 63.5 us against 55.4 us for the single-SM ping-pong kernel, so the
// ping-pong kernel stays the default.
static int g_attn_cp = [] {
    const char* e = std::getenv("CSD_ATTN_CP");
    return e ? std::atoi(e) : 0;
}();

bool attn_cp_supported(const AttnTcArgs& a) {
    return g_attn_cp != 0 && a.idx != nullptr && a.e == E && a.colsum == nullptr && a.row_max == nullptr &&
           a.base != nullptr && a.chunk % 64 == 0 && a.chunk > 128 && a.chunk <= 256 && a.n % a.chunk == 0;
}

cudaError_t attn_cp(const AttnTcArgs& a, cudaStream_t s) {
    const uint64_t cols = a.layout == CSD_LAYOUT_BHNE ? E : (uint64_t)a.heads * E;
    const uint64_t rows = a.layout == CSD_LAYOUT_BHNE ? (uint64_t)(a.batch * a.heads * a.n)
                                                      : (uint64_t)(a.batch * a.n);
    CUtensorMap tq, tb, to;
    if (!make_map_bf16(&tq, a.q, cols, rows, cols, 32) || !make_map_bf16(&tb, a.base, cols, rows, cols, 32) ||
        !make_map_bf16(&to, a.out, cols, rows, cols, 32))
        return cudaErrorInvalidValue;
    CPParams p{};
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
    p.rows = (int)(a.chunk / 2);
    p.order = a.order;
    p.trace = h_cp_trace;
    auto al = [](uint32_t v) { return (v + 1023u) & ~1023u; };
    const uint32_t xbytes = 2u * (uint32_t)p.rows * 128u;
    const uint32_t fixed = 2 * kQBuf + al(xbytes) + 1024 + 1024;  // Q x2, X, barriers, alignment
    p.ns = (int)std::min<uint32_t>(kMaxStages, (kMaxSmem - fixed) / (kKHalf + kVHalf));
    if (p.ns < 2) return cudaErrorNotSupported;
    p.off_k = 2 * kQBuf;
    p.off_v = p.off_k + p.ns * kKHalf;
    p.off_x = p.off_v + p.ns * kVHalf;
    p.x_strip = (uint32_t)p.rows * 128u;
    p.off_bar = al(p.off_x + xbytes);
    const uint32_t smem_bytes = p.off_bar + 512 + 1024;  // + alignment slack of the dynamic base
    if (smem_bytes > kMaxSmem) return cudaErrorNotSupported;
    static const int poly = [] {
        const char* e = std::getenv("CSD_CP_POLY");
        return e ? std::atoi(e) : 0;
    }();
    auto kern = poly == 4 ? k_attn_cp<4> : k_attn_cp<0>;
    cudaError_t err = ensure_smem_attr(kern, (int)kMaxSmem);
    if (err != cudaSuccess) return err;
    const int npairs = (int)std::min<int64_t>(p.items, sm_count() / 2);
    return launch_ex_pdl(1, kern, dim3(2u * (unsigned)npairs), dim3(kThreads), smem_bytes, s, 2, tq, tb, to, p);
}

}  // namespace dev
}  // namespace csd

// Debug only: clock64 timeline of the first kCPTraceCtas CTAs (4 x 2048 uint64; null: off).
extern "C" int csd_debug_set_attn_cp_trace(void* dev_buf) {
    csd::dev::h_cp_trace = static_cast<uint64_t*>(dev_buf);
    return 0;
}

// Debug / test only: route eligible sparse-delta attention launches to the CTA-pair kernel
// (1) or to the ping-pong kernel (0).
extern "C" int csd_debug_set_attn_cp(int on) {
    csd::dev::g_attn_cp = on;
    return 0;
}
