// attn_tc.cu — column-sparse attention on tcgen05 (CSD_MODE_PROD).
//
// Replaces sparse_delta_attention (attention.cpp:147-194), dense_attention
// (:59-74) and the dense-step column sums (:76-145) with ONE kernel family.
//
// Work item = (b, h, query chunk c); Q_c is NT = 1 or 2 M-tiles of 128 rows (c = 192
// uses 2 tiles, 64 idle rows); keys are the chunk's index list (sparse) or all N keys
// (dense baseline / dense step).  Per 128-key block j:
//   producer warp : TMA gather4 of the selected K and V rows (4 rows per instruction,
//                   two 64-column 128B-swizzled strips at E = 128) into a 2-deep ring —
//                   or plain TMA tiles in dense mode;
//   MMA thread    : S_t = Q_t K_j^T  (tcgen05.mma M128 N128 K16, fp32 in TMEM), then
//                   O_t += P_t V_j with P_t read straight from TMEM (TS form; V is the
//                   MN-major smem operand).  The two tiles ping-pong: S_0(j+1) is issued
//                   right after PV_0(j), so tile 0's MMAs overlap tile 1's softmax.
//   softmax warps : one thread per query row (TMEM lane); online softmax over the
//                   SUBSET with lazy rescaling (only when the row max grows by > 2^8),
//                   P_t written back as bf16 over the first 64 columns of S_t;
//                   dense step: chunk column sums with stale stats (warp transpose-reduce).
//   Epilogue: out = base + scale * O / l (the cache update O = O_cache + delta,
//   north_star item 5; base prefetched while the last P·V runs) and row max / exp-sum.
//
// TMEM: S_t (and P_t aliased) at columns [128 t, 128 t + 128); O_t at [128 NT + E t, +E).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <string>

#include "common.cuh"
#include "kernels.h"
#include "launch_util.h"
#include "tc_common.cuh"

namespace csd {
namespace dev {

using namespace csd::tc;

// Debug timeline (scripts/attn_trace.py): when set, CTAs < kTraceCtas record SM clock64()
// stamps at fixed slots (start, Q / K / V issue, S issue, softmax and epilogue phases).
// The buffers travel in the kernel parameters (constant bank): an untraced launch pays a
// uniform predicate per trace point, not a global load on the softmax's critical path.
constexpr int kTraceCtas = 8, kTraceSlots = 1024;
static uint64_t* h_attn_trace = nullptr;  // host-side settings (csd_debug_set_attn_*)
static uint64_t* h_attn_span = nullptr;
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define ATTN_TRACE(slot)                                                                  \
    do {                                                                                  \
        uint64_t* tr_ = p.trace;                                                          \
        if (tr_ != nullptr && blockIdx.x < kTraceCtas && (slot) < kTraceSlots)            \
            tr_[blockIdx.x * kTraceSlots + (slot)] = clock64();                           \
    } while (0)

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

// Shared memory (runtime offsets in AttnParams, 1 KB-aligned regions):
//   [Q: tile t strips of round_up(rows_t, 64) rows][X: staged base tile (sparse with base,
//   chunk <= 192) or the colsum partials][K ring 2 x kKV][V ring 2 x kKV][row-half exchange][bars]
// Q comes first: an M-tile with fewer than 128 live rows reads its 128 MMA rows past the end
// of its strip (into the next strip / X) — dead rows whose P is never used.
template <int E, int NT>
struct AttnLayout {
    static constexpr int kHalves = E / 64;
    static constexpr uint32_t kStrip = 128 * 128;  // 128 rows x 128 B
    static constexpr uint32_t kKV = kHalves * kStrip;  // one K or V block
    static constexpr uint32_t kCsBytes = 2 * 4 * NT * 128 * 4;  // colsum partials [2][NT][4][128]
    static constexpr uint32_t kXchBytes = 2 * 128 * 2 * 4;       // row-half exchange [2][128][2]
    // warpgroup 0: warp 0 (Q / dense K-V TMA, staged-base I/O), warp 1 (MMA), warps 2-3
    // (K/V row copies); warpgroups 1-2: 8 softmax warps, two per TMEM lane quadrant, each
    // owning 64 of a row's 128 key columns; warpgroup 3: four more K/V copy warps.
    static constexpr uint32_t kThreads = 128 + 256 + 128;
    // sparse K/V rows are staged by cp.async from 6 copy warps (warps 2, 3, 12-15): 16 threads
    // per 256-byte row, 16-byte pieces written straight into the 128B-swizzled strips
    static constexpr int kCopyThreads = 192;
    static constexpr uint32_t kTmemCols = (NT * 128 + NT * E) <= 256 ? 256 : 512;
    static constexpr uint32_t kMaxSmem = 227 * 1024;
};

struct AttnParams {
    int stage_base;          // base tile staged in smem region X by TMA (epilogue in smem)
    uint32_t off_x, off_k, off_v, off_xch, off_bar;  // smem region offsets
    uint32_t q_off[2], q_strip[2];  // per M-tile: Q region offset, bytes per 64-column strip
    int q_rows[2];           // per M-tile: Q rows loaded (multiple of 64)
    uint32_t x_strip;        // staged base: bytes per 64-column strip
    const int32_t* idx;
    const int32_t* counts;
    int64_t k_max;
    const __nv_bfloat16* base;
    __nv_bfloat16* out;
    float scale;
    float* row_max;
    float* exp_sum;
    const float* prev_m;
    const float* prev_l;
    float* colsum;
    int layout;
    int heads, n, chunk, chunks, items;
    int cs_chunk, cs_chunks;  // colsum chunking when it differs from the item rows (else 0)
    const __nv_bfloat16* kp;  // raw K / V (the cp.async row gather)
    const __nv_bfloat16* vp;
    int cp_async;             // sparse K/V staging: 1 = cp.async copy warps, 0 = TMA gather4
    uint64_t* trace;          // debug timeline (null: off)
    uint64_t* span;           // debug per-CTA [start, end] globaltimer (null: off)
    float qk_scale_log2;  // log2(e) / sqrt(E)
};

__device__ __forceinline__ int64_t tok_elem_off(int layout, int64_t b, int64_t h, int64_t tok,
                                                int heads, int n, int e) {
    return layout == CSD_LAYOUT_BHNE ? (((b * heads + h) * (int64_t)n) + tok) * e
                                     : ((b * (int64_t)n + tok) * heads + h) * e;
}

template <int E, int NT>
__global__ void __launch_bounds__(AttnLayout<E, NT>::kThreads, 1)
k_attn_tc(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
          const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_kg,
          const __grid_constant__ CUtensorMap tm_vg, const __grid_constant__ CUtensorMap tm_b,
          const __grid_constant__ CUtensorMap tm_o, const AttnParams p) {
    using L = AttnLayout<E, NT>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_u32 = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);

    // Persistent: CTA b processes items b, b + grid, ...  Every role walks the same item
    // sequence and skips count-0 items identically, so ring / barrier phases run on two
    // counters shared by all roles: `li` (live items) and `gb` (key blocks).
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool dense = p.idx == nullptr;
    const int items = p.items;
    if (threadIdx.x == 0) ATTN_TRACE(0);
    if (threadIdx.x == 0 && p.span != nullptr) p.span[2 * blockIdx.x] = globaltimer_ns();

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
    uint64_t* bar_q = bars + 0;
    uint64_t* bar_kf = bars + 1;   // [2]
    uint64_t* bar_ke = bars + 3;   // [2]
    uint64_t* bar_vf = bars + 5;   // [2]
    uint64_t* bar_ve = bars + 7;   // [2]
    uint64_t* bar_s = bars + 9;    // [NT]
    uint64_t* bar_p = bars + 11;   // [NT]
    uint64_t* bar_o = bars + 13;
    uint64_t* bar_qe = bars + 14;  // Q buffer free (all S MMAs of the item done)
    uint64_t* bar_bf = bars + 17;   // staged base tile of the current live item landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);
    uint64_t* bar_xc = bars + 19;   // every live softmax warp combined its rows into X
    uint8_t* const sq = smem;
    uint8_t* const sx = smem + p.off_x;
    uint8_t* const sk = smem + p.off_k;
    uint8_t* const sv = smem + p.off_v;
    if (threadIdx.x == 0) {
        // the host sizes the request without alignment slack (the 227 KB budget is tight)
        if ((raw_u32 & 1023u) != 0) __trap();
        mbar_init(bar_q, 1);
        // cp.async staging: one cp.async.mbarrier arrival per copy thread per block;
        // TMA (tiles / gather4): one expect_tx arrival
        const uint32_t fill = (!dense && p.cp_async) ? (uint32_t)L::kCopyThreads : 1u;
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar_kf + i, fill);
            mbar_init(bar_ke + i, 1);
            mbar_init(bar_vf + i, fill);
            mbar_init(bar_ve + i, 1);
        }
        for (int t = 0; t < NT; ++t) {
            mbar_init(bar_s + t, 1);
            mbar_init(bar_p + t, 256);  // every softmax thread (dead rows write P = 0)
        }
        mbar_init(bar_o, 1);
        mbar_init(bar_qe, 1);
        mbar_init(bar_bf, 1);
        mbar_init(bar_xc, 8);  // one arrival per softmax warp
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<L::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) ATTN_TRACE(1);
    const bool cpa = !dense && p.cp_async;
    // next live (count > 0) item of this CTA at or after `from`
    auto next_live = [&](int from, int& cnt_out) -> int {
        int x = from;
        cnt_out = 0;
        for (; x < items; x += gridDim.x) {
            cnt_out = dense ? p.n : p.counts[x];
            if (cnt_out > 0) break;
        }
        return x;
    };
    // staged base tile of `item` -> region X (64-row TMA boxes, 128B-swizzled strips)
    auto issue_base = [&](int it) {
        const int bh2 = it / p.chunks;
        const int rb2 = p.layout == CSD_LAYOUT_BHNE ? bh2 * p.n : (bh2 / p.heads) * p.n;
        const int cl2 = p.layout == CSD_LAYOUT_BHNE ? 0 : (bh2 % p.heads) * E;
        const int nbox = (p.chunk + 63) >> 6;
        fence_proxy_async_smem();  // prior generic reads of X before the async-proxy refill
        mbar_arrive_expect_tx(bar_bf, (uint32_t)(L::kHalves * nbox) * 8192u);
        for (int hf = 0; hf < L::kHalves; ++hf)
            for (int bx = 0; bx < nbox; ++bx)
                tma_load_2d(&tm_b, bar_bf, sx + hf * p.x_strip + bx * 8192, cl2 + hf * 64,
                            rb2 + (it % p.chunks) * p.chunk + bx * 64);
    };
    // staged-base I/O thread (warp 0 lane 31): per live item, base
    // tile in, then -- once every softmax warp has combined its rows in place -- the out tile
    // out by TMA store, then the next item's base tile in
    auto io_thread = [&]() {
        int nc = 0;
        int it = next_live(blockIdx.x, nc);
        if (it < items) issue_base(it);
        uint32_t li = 0;
        while (it < items) {
            const int bh2 = it / p.chunks, c2 = it % p.chunks;
            const int rb = p.layout == CSD_LAYOUT_BHNE ? bh2 * p.n : (bh2 / p.heads) * p.n;
            const int cl = p.layout == CSD_LAYOUT_BHNE ? 0 : (bh2 % p.heads) * E;
            const int nx = next_live(it + gridDim.x, nc);
            mbar_wait(bar_xc, li & 1);
            fence_proxy_async_smem();
            const int nbox = (p.chunk + 63) >> 6;
            for (int hf = 0; hf < L::kHalves; ++hf)
                for (int bx = 0; bx < nbox; ++bx)
                    tma_store_2d(&tm_o, sx + hf * p.x_strip + bx * 8192, cl + hf * 64,
                                 rb + c2 * p.chunk + bx * 64);
            bulk_commit();
            bulk_wait_read0();  // X read out before it is refilled
            if (nx < items) issue_base(nx);
            it = nx;
            ++li;
        }
        bulk_wait0();  // the last out tile has landed before the CTA exits
    };
    // ---------------------------------------------------------------- producers
    // Every loader walks the same live-item / key-block sequence (counters li, gb).
    // Q tiles (all modes) and the dense K/V tiles: warp 0 lane 0, plain TMA.
    auto q_loader = [&]() {
        tma_prefetch_desc(&tm_q);
        if (dense) {
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_v);
        }
        uint32_t gb = 0, li = 0;
        for (int item = blockIdx.x; item < items; item += gridDim.x) {
            const int cnt = dense ? p.n : p.counts[item];
            if (cnt == 0) continue;
            const int c = item % p.chunks, bh = item / p.chunks;
            const int b = bh / p.heads, h = bh % p.heads;
            const int row_base = p.layout == CSD_LAYOUT_BHNE ? bh * p.n : b * p.n;
            const int col0 = p.layout == CSD_LAYOUT_BHNE ? 0 : h * E;
            const int nblk = (cnt + 127) / 128;
            if (li > 0) mbar_wait(bar_qe, (li - 1) & 1);  // previous item's S MMAs done
            ATTN_TRACE(2 + li);
            mbar_arrive_expect_tx(bar_q, (uint32_t)(L::kHalves * (p.q_rows[0] + (NT > 1 ? p.q_rows[1] : 0))) * 128u);
            for (int t = 0; t < NT; ++t)
                for (int hf = 0; hf < L::kHalves; ++hf)
                    for (int bx = 0; bx < p.q_rows[t] / 64; ++bx)  // 64-row boxes
                        tma_load_2d(&tm_q, bar_q, sq + p.q_off[t] + hf * p.q_strip[t] + bx * 8192,
                                    col0 + hf * 64, row_base + c * p.chunk + t * 128 + bx * 64);
            if (dense) {
                for (int j = 0; j < nblk; ++j, ++gb) {
                    const int s = gb & 1;
                    if (gb >= 2) mbar_wait(bar_ke + s, ((gb >> 1) - 1) & 1);
                    ATTN_TRACE(16 + gb);
                    mbar_arrive_expect_tx(bar_kf + s, L::kKV);
                    for (int hf = 0; hf < L::kHalves; ++hf)
                        tma_load_2d(&tm_k, bar_kf + s, sk + s * L::kKV + hf * L::kStrip, col0 + hf * 64,
                                    row_base + j * 128);
                    if (gb >= 2) mbar_wait(bar_ve + s, ((gb >> 1) - 1) & 1);
                    mbar_arrive_expect_tx(bar_vf + s, L::kKV);
                    for (int hf = 0; hf < L::kHalves; ++hf)
                        tma_load_2d(&tm_v, bar_vf + s, sv + s * L::kKV + hf * L::kStrip, col0 + hf * 64,
                                    row_base + j * 128);
                    ATTN_TRACE(48 + gb);
                }
            }
            ++li;
        }
    };
    // Sparse K/V rows by TMA tile::gather4 (4 rows per instruction, one instruction per
    // 64-column strip), spread over three warps (lane % 3 == pw).
    auto gather4_loader = [&](int pw) {
        const bool mine = (lane % 3) == pw;
        if (pw == 0 && lane == 0) {
            tma_prefetch_desc(&tm_kg);
            tma_prefetch_desc(&tm_vg);
        }
        uint32_t gb = 0;
        for (int item = blockIdx.x; item < items; item += gridDim.x) {
            const int cnt = p.counts[item];
            if (cnt == 0) continue;
            const int bh = item / p.chunks;
            const int b = bh / p.heads, h = bh % p.heads;
            const int row_base = p.layout == CSD_LAYOUT_BHNE ? bh * p.n : b * p.n;
            const int col0 = p.layout == CSD_LAYOUT_BHNE ? 0 : h * E;
            const int nblk = (cnt + 127) / 128;
            const int32_t* ids = p.idx + (int64_t)item * p.k_max;
            for (int j = 0; j < nblk; ++j, ++gb) {
                const int s = gb & 1;
                int32_t rows[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    int r = j * 128 + lane * 4 + i;
                    r = r < cnt ? r : cnt - 1;  // pad with a valid row (masked in softmax)
                    rows[i] = row_base + __ldg(ids + r);
                }
                if (gb >= 2) mbar_wait(bar_ke + s, ((gb >> 1) - 1) & 1);
                if (pw == 0 && lane == 0) mbar_arrive_expect_tx(bar_kf + s, L::kKV);
                if (mine)
                    for (int hf = 0; hf < L::kHalves; ++hf)
                        tma_gather4(&tm_kg, bar_kf + s, sk + s * L::kKV + hf * L::kStrip + lane * 512,
                                    col0 + hf * 64, rows[0], rows[1], rows[2], rows[3]);
                if (gb >= 2) mbar_wait(bar_ve + s, ((gb >> 1) - 1) & 1);
                if (pw == 0 && lane == 0) mbar_arrive_expect_tx(bar_vf + s, L::kKV);
                if (mine)
                    for (int hf = 0; hf < L::kHalves; ++hf)
                        tma_gather4(&tm_vg, bar_vf + s, sv + s * L::kKV + hf * L::kStrip + lane * 512,
                                    col0 + hf * 64, rows[0], rows[1], rows[2], rows[3]);
            }
        }
    };
    // Sparse K/V rows by cp.async (LSU path, ~2.5x gather4's per-SM rate): copy thread ct
    // owns the fixed 16-byte pieces ct + kCopyThreads * i of every block (16 pieces per
    // 256-byte row, consecutive threads on one row), written straight into the 128B-swizzled
    // strips; rows past the chunk's count are zero-filled (src-size 0: no global read), so
    // the dead key columns of the last block hold finite zeros.  One
    // cp.async.mbarrier.arrive.noinc per thread per K (V) block completes the fill barrier.
    auto copy_loader = [&](int ct) {
        // kCopyThreads = 12 x 16: thread ct always copies 16-byte column piece c16 = ct % 16
        // of rows r0 + 12 i (r0 = ct / 16), i.e. the same smem column slot in every block
        static_assert(L::kCopyThreads % (E / 8) == 0, "copy threads per row");
        constexpr int kRowStep = L::kCopyThreads / (E / 8);
        constexpr int kRows = (128 + kRowStep - 1) / kRowStep;
        const int c16 = ct % (E / 8), r0 = ct / (E / 8);
        const uint32_t cbase = (uint32_t)(c16 >> 3) * L::kStrip;
        const int64_t rs = p.layout == CSD_LAYOUT_BHNE ? E : (int64_t)p.heads * E;  // row stride
        const uint32_t sK = smem_u32(sk), sV = smem_u32(sv);
        uint32_t gb = 0;
        for (int item = blockIdx.x; item < items; item += gridDim.x) {
            const int cnt = p.counts[item];
            if (cnt == 0) continue;
            const int bh = item / p.chunks;
            const int b = bh / p.heads, h = bh % p.heads;
            const int64_t o0 = tok_elem_off(p.layout, b, h, 0, p.heads, p.n, E) + c16 * 8;
            const __nv_bfloat16* kb = p.kp + o0;
            const __nv_bfloat16* vb = p.vp + o0;
            const int nblk = (cnt + 127) / 128;
            const int32_t* ids = p.idx + (int64_t)item * p.k_max;
            for (int j = 0; j < nblk; ++j, ++gb) {
                const int s = gb & 1;
                int32_t id[kRows];
#pragma unroll
                for (int i = 0; i < kRows; ++i) {
                    const int r = j * 128 + r0 + kRowStep * i;
                    id[i] = (r0 + kRowStep * i < 128 && r < cnt) ? __ldg(ids + r) : -1;
                }
                if (gb >= 2) mbar_wait(bar_ke + s, ((gb >> 1) - 1) & 1);
#pragma unroll
                for (int i = 0; i < kRows; ++i) {
                    const uint32_t row = (uint32_t)(r0 + kRowStep * i);
                    if (row < 128u)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                                         sK + s * L::kKV + cbase + sw128_offset(row, (uint32_t)(c16 & 7))),
                                     "l"(kb + (id[i] >= 0 ? (int64_t)id[i] * rs : 0)), "r"(id[i] >= 0 ? 16u : 0u)
                                     : "memory");
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar_kf + s)) : "memory");
                if (gb >= 2) mbar_wait(bar_ve + s, ((gb >> 1) - 1) & 1);
#pragma unroll
                for (int i = 0; i < kRows; ++i) {
                    const uint32_t row = (uint32_t)(r0 + kRowStep * i);
                    if (row < 128u)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                                         sV + s * L::kKV + cbase + sw128_offset(row, (uint32_t)(c16 & 7))),
                                     "l"(vb + (id[i] >= 0 ? (int64_t)id[i] * rs : 0)), "r"(id[i] >= 0 ? 16u : 0u)
                                     : "memory");
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar_vf + s)) : "memory");
            }
        }
    };
    // Registers go to the softmax warpgroups (1, 2): 4 x 128 x 128 at launch = 2 x 128 x 72 +
    // 2 x 128 x 184.  Each role branch starts with its warpgroup's setmaxnreg so the
    // register budget of the code below it is known to ptxas.
    if (warp < 4 || warp >= 12) {
    regs_dec<72>();
    if (warp == 0) {
        if (lane == 0) q_loader();
        else if (lane == 31 && p.stage_base) io_thread();
    } else if (warp == 2 || warp == 3 || warp >= 12) {
        if (!dense) {
            if (p.cp_async) copy_loader(warp < 4 ? (warp - 2) * 32 + lane : 64 + (warp - 12) * 32 + lane);
            else if (warp <= 12) gather4_loader(warp == 12 ? 2 : warp - 2);
        }
    } else {
        // ------------------------------------------------------------ MMA issuer (warp 1)
        // The whole warp walks the schedule so the descriptors are warp-uniform (uniform
        // registers, no per-MMA broadcast); lane 0 (elect.sync's leader) issues every MMA
        // and commit, so the commits track that lane's MMAs.
        {
            constexpr uint32_t idS = idesc_bf16(128, 128, false, false);
            constexpr uint32_t idO = idesc_bf16(128, E, false, true);
            const uint32_t sQ = smem_u32(sq), sK = smem_u32(sk);
            const uint32_t sV = smem_u32(sv);
            auto commit = [&](uint64_t* b) {
                if (elect_one()) mma_commit(b);
                __syncwarp();
            };
            auto issue_s = [&](int t, uint32_t g) {  // S_t = Q_t K_g^T
                const uint32_t kb = sK + (g & 1) * L::kKV;
                uint64_t da[E / 16], db[E / 16];
#pragma unroll
                for (int kk = 0; kk < E / 16; ++kk) {
                    da[kk] = desc_kmajor_sw128(sQ + p.q_off[t] + (kk / 4) * p.q_strip[t] + (kk % 4) * 32);
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
                        mma_bf16_ts(tmem + NT * 128 + t * E, tmem + t * 128 + kk * 8, dv[kk], idO,
                                    (acc || kk > 0) ? 1u : 0u);
                }
                __syncwarp();
            };
            uint32_t gb = 0, li = 0;
            for (int item = blockIdx.x; item < items; item += gridDim.x) {
                const int cnt = dense ? p.n : p.counts[item];
                if (cnt == 0) continue;
                const int nblk = (cnt + 127) / 128;
                // S_t(0) may overwrite S_t / P_t of the previous item: PV_t(last) was issued
                // earlier and tcgen05 MMAs of one thread execute in order
                mbar_wait(bar_q, li & 1);
                ATTN_TRACE(8 + li);
                mbar_wait(bar_kf + (gb & 1), (gb >> 1) & 1);
                if (cpa) fence_proxy_async_smem();  // cp.async (generic proxy) -> tcgen05 reads
                tc_fence_after();
                ATTN_TRACE(80 + gb);
                for (int t = 0; t < NT; ++t) issue_s(t, gb);
                commit(bar_ke + (gb & 1));
                if (nblk == 1) commit(bar_qe);
                for (int j = 0; j < nblk; ++j) {
                    const uint32_t g = gb + j;
                    const bool more = j + 1 < nblk;
                    for (int t = 0; t < NT; ++t) {
                        // P_t(j) in TMEM and O_t rescaled; for j = 0 this also orders the
                        // previous item's epilogue reads of O_t (same warps, program order)
                        mbar_wait(bar_p + t, g & 1);
                        if (t == 0) {
                            mbar_wait(bar_vf + (g & 1), (g >> 1) & 1);
                            if (cpa) fence_proxy_async_smem();
                            ATTN_TRACE(832 + (g & 63));
                        }
                        tc_fence_after();
                        ATTN_TRACE(640 + 64 * t + (g & 63));
                        issue_pv(t, g, j > 0);
                        if (t == NT - 1) commit(bar_ve + (g & 1));
                        if (more) {
                            if (t == 0) {
                                mbar_wait(bar_kf + ((g + 1) & 1), ((g + 1) >> 1) & 1);
                                if (cpa) fence_proxy_async_smem();
                                tc_fence_after();
                                ATTN_TRACE(80 + g + 1);
                                ATTN_TRACE(768 + ((g + 1) & 63));
                            }
                            ATTN_TRACE(512 + 64 * t + ((g + 1) & 63));
                            issue_s(t, g + 1);  // in-order after PV_t(j): P_t consumed first
                            if (t == NT - 1) {
                                commit(bar_ke + ((g + 1) & 1));
                                if (j + 2 == nblk) commit(bar_qe);
                            }
                        }
                    }
                }
                commit(bar_o);
                gb += nblk;
                ++li;
            }
        }
    }
    } else {
        regs_inc<184>();
        // ------------------------------------------------------------ softmax / epilogue
        // 8 warps: warp 4 + 4 hf + quad owns TMEM lane quadrant `quad` (rows quad * 32 + lane
        // of every M-tile) and key columns [64 hf, 64 hf + 64) of each S block.  The two
        // halves of a row meet in smem (row max per block, row sum per item) behind a
        // 64-thread named barrier per quadrant.  All 8 warps walk the M-tiles one after the
        // other, so tile t's exponentials run at the full MUFU rate while the MMA pipe works
        // on tile 1 - t (P.V then the next S).
        const int sw = warp - 4;  // 0 .. 7
        const int hf = sw >> 2, quad = sw & 3;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        float* cs_part = reinterpret_cast<float*>(sx);  // [2][NT][4][128]
        float* xch = reinterpret_cast<float*>(smem + p.off_xch);  // [2][128][2]
        const bool do_cs = p.colsum != nullptr;
        const float sl2 = p.qk_scale_log2;
        const int qbar = 2 + quad;  // the quadrant's two warps
        constexpr int kOc = E / 64;  // 32-column O groups per half
        uint32_t gb = 0, li = 0;
        for (int item = blockIdx.x; item < items; item += gridDim.x) {
            const int cnt = dense ? p.n : p.counts[item];
            const int c = item % p.chunks, bh = item / p.chunks;
            const int b = bh / p.heads, h = bh % p.heads;
            if (cnt == 0) {  // pass base through (attention.cpp:169)
                if (p.base != p.out && p.base != nullptr) {
                    for (int r = threadIdx.x - 128; r < p.chunk * (E / 8); r += 256) {
                        const int row = r / (E / 8), v8 = r % (E / 8);
                        const int64_t off = tok_elem_off(p.layout, b, h, (int64_t)c * p.chunk + row,
                                                         p.heads, p.n, E) + v8 * 8;
                        *reinterpret_cast<uint4*>(p.out + off) =
                            *reinterpret_cast<const uint4*>(p.base + off);
                    }
                }
                continue;
            }
            const int nblk = (cnt + 127) / 128;
            float m_run[NT], m_true[NT], l_run[NT], mpl[NT], inv_lp[NT];
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                m_run[t] = -INFINITY;
                m_true[t] = -INFINITY;
                l_run[t] = 0.f;
                mpl[t] = 0.f;
                inv_lp[t] = 0.f;
                const int crow = t * 128 + quad * 32 + lane;
                if (do_cs && crow < p.chunk) {
                    const int64_t si = (int64_t)bh * p.n + (int64_t)c * p.chunk + crow;
                    mpl[t] = p.prev_m[si] * kLog2e;
                    inv_lp[t] = 1.0f / p.prev_l[si];
                }
            }
            for (int j = 0; j < nblk; ++j) {
                const uint32_t g = gb + j;
                const int ncols = min(128, cnt - j * 128);
                const int nh = min(64, max(0, ncols - 64 * hf));  // live columns of this half
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    const int crow = t * 128 + quad * 32 + lane;
                    const bool row_ok = crow < p.chunk;
                    const bool warp_ok = t * 128 + quad * 32 < p.chunk;  // same for both halves
                    const uint32_t tS = tmem + lane_off + t * 128;
                    const uint32_t tO = tmem + lane_off + NT * 128 + t * E;
                    mbar_wait(bar_s + t, g & 1);
                    tc_fence_after();
                    if (lane == 0 && sw == 0) ATTN_TRACE(144 + g);
                    if (lane == 0 && quad == 0 && hf == 0) ATTN_TRACE(256 + 64 * t + (g & 63));
                    if (warp_ok) {
                        // this half's 64 S columns (2 TMEM loads in flight, one wait)
                        const bool full = nh == 64 && __all_sync(0xffffffffu, row_ok);
                        uint32_t sr[64];
                        if (nh > 0) {  // uniform
                            tmem_ld32(tS + hf * 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
                            tmem_ld32(tS + hf * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
                            tmem_ld_wait();
                        }
                        if (!full) {
#pragma unroll
                            for (int i = 0; i < 64; ++i)
                                if (i >= nh) sr[i] = __float_as_uint(-INFINITY);
                        }
                        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                        for (int i = 0; i < 64; i += 8)
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                mx4[u] = fmax3(mx4[u], __uint_as_float(sr[i + 2 * u]),
                                               __uint_as_float(sr[i + 2 * u + 1]));
                        const float mloc = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
                        // row max across the halves; slot t (NT = 2: the other tile's exchange
                        // sits between two uses) or block parity (NT = 1)
                        float* xr = xch + ((NT == 2 ? t : (int)(g & 1)) * 128 + quad * 32 + lane) * 2;
                        xr[hf] = mloc;
                        named_bar_sync(qbar, 64);
                        const float mraw = fmaxf(mloc, xr[hf ^ 1]);
                        const float mx = row_ok ? mraw * sl2 : -INFINITY;  // sl2 > 0: max commutes
                        m_true[t] = fmaxf(m_true[t], mx);
                        const bool need = mx > m_run[t] + kRescaleThreshold;
                        const float alpha = need ? ex2_approx(m_run[t] - mx) : 1.0f;
                        if (need) {
                            m_run[t] = mx;
                            l_run[t] *= alpha;
                        }
                        if (j > 0 && __any_sync(0xffffffffu, need)) {  // PV_t(j-1) done (bar_s order)
#pragma unroll 1
                            for (int oc = 0; oc < kOc; ++oc) {
                                uint32_t r[32];
                                tmem_ld32(tO + (hf * kOc + oc) * 32, r);
                                tmem_ld_wait();
#pragma unroll
                                for (int i = 0; i < 32; ++i)
                                    r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                                tmem_st32(tO + (hf * kOc + oc) * 32, r);
                            }
                        }
                        const float w = do_cs ? ex2_approx(m_run[t] - mpl[t]) * inv_lp[t] : 0.f;
                        const float neg_m = row_ok ? -m_run[t] : -INFINITY;  // dead rows -> p = 0
                        const float2 sl2v = make_float2(sl2, sl2), nm2 = make_float2(neg_m, neg_m);
                        float2 part0 = make_float2(0.f, 0.f), part1 = make_float2(0.f, 0.f);
#pragma unroll
                        for (int cc = 0; cc < 2; ++cc) {
                            float* csp = cs_part + ((((g & 1) * NT + t) * 4 + quad) * 128) + hf * 64 + cc * 32;
                            if (cc * 32 >= nh) {  // uniform: a fully masked group contributes P = 0
                                uint32_t pk[16];
#pragma unroll
                                for (int q = 0; q < 16; ++q) pk[q] = 0u;
                                tmem_st16(tS + hf * 32 + cc * 16, pk);
                                if (do_cs) csp[lane] = 0.f;
                                continue;
                            }
                            float pv[32];
                            // 2^(S*scale - m) with paired FFMA2 / FADD2 (two row sums in flight)
#pragma unroll
                            for (int q = 0; q < 16; ++q) {
                                const float2 x = make_float2(__uint_as_float(sr[cc * 32 + 2 * q]),
                                                             __uint_as_float(sr[cc * 32 + 2 * q + 1]));
                                const float2 y = __ffma2_rn(x, sl2v, nm2);
                                float2 e;
                                e.x = ex2_approx(y.x);
                                e.y = ex2_approx(y.y);
                                pv[2 * q] = e.x;
                                pv[2 * q + 1] = e.y;
                                if (q & 1) part1 = __fadd2_rn(part1, e);
                                else part0 = __fadd2_rn(part0, e);
                            }
                            // P_t (bf16 pairs) over S_t columns [32 hf + 16 cc, +16): both halves'
                            // S loads completed before the exchange barrier
                            uint32_t pk[16];
#pragma unroll
                            for (int q = 0; q < 16; ++q) pk[q] = pack_bf16x2(pv[2 * q], pv[2 * q + 1]);
                            tmem_st16(tS + hf * 32 + cc * 16, pk);
                            if (do_cs) {
                                // transpose-reduce the warp's 32 x 32 block of w * p on packed
                                // f16 column pairs (16 shuffles instead of 31; the sums only
                                // rank keys for the top-k): after the rounds over lane bits
                                // 4..1 lane l holds columns (l & ~1, l | 1) over half the
                                // lanes, the last exchange adds the other half
                                uint32_t hp[16];
                                const float2 w2 = make_float2(w, w);
#pragma unroll
                                for (int q = 0; q < 16; ++q)
                                    hp[q] = pack_f16x2(__fmul2_rn(make_float2(pv[2 * q], pv[2 * q + 1]), w2));
#pragma unroll
                                for (int wd = 16, hw = 8; wd >= 2; wd >>= 1, hw >>= 1) {
                                    const bool upper = (lane & wd) != 0;
#pragma unroll
                                    for (int i = 0; i < hw; ++i) {
                                        const uint32_t send = upper ? hp[i] : hp[i + hw];
                                        const uint32_t keep = upper ? hp[i + hw] : hp[i];
                                        hp[i] = hadd2_u32(keep, __shfl_xor_sync(0xffffffffu, send, wd));
                                    }
                                }
                                const float2 tot = unpack_f16x2(hadd2_u32(hp[0], __shfl_xor_sync(0xffffffffu, hp[0], 1)));
                                csp[lane] = (lane & 1) ? tot.y : tot.x;
                            }
                        }
                        const float2 part = __fadd2_rn(part0, part1);
                        l_run[t] += part.x + part.y;
                    } else {
                        // rows past the chunk: zero P so the padded MMA rows stay finite
                        uint32_t pk[16];
#pragma unroll
                        for (int q = 0; q < 16; ++q) pk[q] = 0u;
                        tmem_st16(tS + hf * 32, pk);
                        tmem_st16(tS + hf * 32 + 16, pk);
                    }
                    tmem_st_wait();
                    tc_fence_before();
                    mbar_arrive(bar_p + t);
                    if (lane == 0 && sw == 0) ATTN_TRACE(168 + g);
                    if (lane == 0 && quad == 0 && hf == 0) ATTN_TRACE(384 + 64 * t + (g & 63));
                }
                if (do_cs) {
                    named_bar_sync(1, 256);
                    const int st = sw * 32 + lane;
                    if (st < 128 && st < ncols && p.cs_chunk == 0) {
                        float s = 0.f;
                        for (int t = 0; t < NT; ++t)
                            for (int qd = 0; qd < 4; ++qd)
                                if (t * 128 + qd * 32 < p.chunk)
                                    s += cs_part[(((g & 1) * NT + t) * 4 + qd) * 128 + st];
                        p.colsum[((int64_t)bh * p.chunks + c) * p.n + j * 128 + st] = s;
                    } else if (st < 128 && st < ncols) {
                        // item rows != colsum chunk (256-row items over, e.g., 192-row chunks):
                        // every 32-row quadrant lies in one chunk and an item touches at most
                        // two; each (chunk, key) gets at most two atomic adds onto a zeroed
                        // output, so the sum is order-independent (a + b == b + a)
                        const int64_t r0 = (int64_t)c * p.chunk;
                        const int64_t c_lo = r0 / p.cs_chunk;
                        float s_lo = 0.f, s_hi = 0.f;
                        bool hi = false;
                        for (int t = 0; t < NT; ++t)
                            for (int qd = 0; qd < 4; ++qd)
                                if (t * 128 + qd * 32 < p.chunk) {
                                    const float vv = cs_part[(((g & 1) * NT + t) * 4 + qd) * 128 + st];
                                    if ((r0 + t * 128 + qd * 32) / p.cs_chunk == c_lo) {
                                        s_lo += vv;
                                    } else {
                                        s_hi += vv;
                                        hi = true;
                                    }
                                }
                        float* cs0 = p.colsum + ((int64_t)bh * p.cs_chunks + c_lo) * p.n + j * 128 + st;
                        atomicAdd(cs0, s_lo);
                        if (hi) atomicAdd(cs0 + p.n, s_hi);
                    }
                }
            }
            // ------------------------------------------------------------ epilogue
            // full row sums: the halves swap partial sums for all tiles at once (the first
            // barrier retires the last block's max exchange, the third this exchange before
            // the next item reuses xch)
            float l_full[NT];
            named_bar_sync(qbar, 64);
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                l_full[t] = l_run[t];
                if (t * 128 + quad * 32 < p.chunk) xch[(t * 128 + quad * 32 + lane) * 2 + hf] = l_run[t];
            }
            named_bar_sync(qbar, 64);
#pragma unroll
            for (int t = 0; t < NT; ++t)
                if (t * 128 + quad * 32 < p.chunk)
                    l_full[t] = l_run[t] + xch[(t * 128 + quad * 32 + lane) * 2 + (hf ^ 1)];
            named_bar_sync(qbar, 64);
            const bool has_base = p.base != nullptr;
            if (p.stage_base) {
                // out = base + scale * O / l (north_star item 5) with the item's base tile
                // already in smem (TMA, issued at the end of the previous item's epilogue):
                // each thread combines its half row in place (bf16, swizzled); the I/O thread
                // stores the tile by TMA.
                mbar_wait(bar_o, li & 1);
                mbar_wait(bar_bf, li & 1);
                tc_fence_after();
                if (lane == 0 && sw == 0) ATTN_TRACE(240 + li);
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    const int crow = t * 128 + quad * 32 + lane;
                    const bool row_ok = crow < p.chunk;
                    if (t * 128 + quad * 32 >= p.chunk) continue;  // uniform per warp
                    const uint32_t tO = tmem + lane_off + NT * 128 + t * E;
                    const float fsc = p.scale / l_full[t];
#pragma unroll
                    for (int o2 = 0; o2 < kOc; ++o2) {
                        const int oc = hf * kOc + o2;
                        uint32_t r[32];
                        tmem_ld32(tO + oc * 32, r);
                        tmem_ld_wait();
                        if (!row_ok) continue;
                        uint8_t* rowp = sx + (oc >> 1) * p.x_strip + crow * 128;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int cidx = (oc & 1) * 4 + q;
                            uint4* ptr = reinterpret_cast<uint4*>(rowp + ((cidx ^ (crow & 7)) << 4));
                            const uint4 bv = *ptr;
                            const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&bv);
                            uint32_t o4[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const float2 f = __bfloat1622float2(b2[u]);
                                o4[u] = pack_bf16x2(fmaf(fsc, __uint_as_float(r[q * 8 + 2 * u]), f.x),
                                                    fmaf(fsc, __uint_as_float(r[q * 8 + 2 * u + 1]), f.y));
                            }
                            *ptr = make_uint4(o4[0], o4[1], o4[2], o4[3]);
                        }
                    }
                    if (row_ok && hf == 0 && p.row_max != nullptr) {
                        const int64_t si = (int64_t)bh * p.n + (int64_t)c * p.chunk + crow;
                        p.row_max[si] = m_true[t] * kLn2;
                        p.exp_sum[si] = l_full[t] * exp2f(m_run[t] - m_true[t]);
                    }
                }
                if (lane == 0 && sw == 0) ATTN_TRACE(232 + li);
                // hand X to the I/O thread (warp 0 lane 31): it stores the out tile by TMA and
                // refills X with the next live item's base tile; the softmax warps go on
                fence_proxy_async_smem();  // this thread's in-place writes -> async proxy
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_xc);
            } else {
                mbar_wait(bar_o, li & 1);
                tc_fence_after();
                if (lane == 0 && sw == 0) ATTN_TRACE(240 + li);
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    const int crow = t * 128 + quad * 32 + lane;
                    const bool row_ok = crow < p.chunk;
                    if (t * 128 + quad * 32 >= p.chunk) continue;  // uniform per warp
                    const uint32_t tO = tmem + lane_off + NT * 128 + t * E;
                    const int64_t tok = (int64_t)c * p.chunk + crow;
                    const int64_t off = tok_elem_off(p.layout, b, h, tok, p.heads, p.n, E);
                    const float inv_l = 1.0f / l_full[t];
#pragma unroll
                    for (int o2 = 0; o2 < kOc; ++o2) {
                        const int oc = hf * kOc + o2;
                        uint32_t r[32];
                        tmem_ld32(tO + oc * 32, r);
                        tmem_ld_wait();
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
                            dp[q] = v;
                        }
                    }
                    if (row_ok && hf == 0 && p.row_max != nullptr) {
                        const int64_t si = (int64_t)bh * p.n + tok;
                        p.row_max[si] = m_true[t] * kLn2;
                        p.exp_sum[si] = l_full[t] * exp2f(m_run[t] - m_true[t]);
                    }
                }
            }
            if (lane == 0 && sw == 0) ATTN_TRACE(248 + li);
            tc_fence_before();  // O reads ordered before the next item's bar_p arrive
            gb += nblk;
            ++li;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0 && p.span != nullptr) p.span[2 * blockIdx.x + 1] = globaltimer_ns();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<L::kTmemCols>(tmem);
    }
}

// ---------------------------------------------------------------------------
// Host side: tensor maps through the driver entry point (no -lcuda needed).
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

// 2-D bf16 map [rows][cols] with row pitch `pitch_elems`, box {64, box_rows}, 128 B swizzle.
bool make_map_bf16(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows,
                   uint64_t pitch_elems, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {pitch_elems * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// General 2-D map: element size 2 (bf16) or 4 (fp32), box {box_cols, box_rows}, the given
// swizzle (box_cols * elem_bytes must equal the swizzle span for the swizzled modes).
bool make_map_2d(CUtensorMap* m, const void* base, int elem_bytes, uint64_t cols, uint64_t rows,
                 uint64_t pitch_elems, uint32_t box_cols, uint32_t box_rows, int swizzle_bytes) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {pitch_elems * (uint64_t)elem_bytes};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                        : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = fn(m, elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                    const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool attn_tc_supported(int64_t e, int64_t chunk) {
    return (e == 64 || e == 128) && chunk >= 1 && chunk <= 256;
}

template <int E, int NT>
static cudaError_t launch_attn(const AttnTcArgs& a, cudaStream_t s) {
    using L = AttnLayout<E, NT>;
    const uint64_t cols = a.layout == CSD_LAYOUT_BHNE ? E : (uint64_t)a.heads * E;
    const uint64_t rows = a.layout == CSD_LAYOUT_BHNE ? (uint64_t)(a.batch * a.heads * a.n)
                                                      : (uint64_t)(a.batch * a.n);
    CUtensorMap tq, tk, tv, tkg, tvg, tb, to;
    if (!make_map_bf16(&tq, a.q, cols, rows, cols, 64) ||
        !make_map_bf16(&to, a.out, cols, rows, cols, 64) ||
        !make_map_bf16(&tb, a.base != nullptr ? a.base : a.q, cols, rows, cols, 64) ||
        !make_map_bf16(&tk, a.k, cols, rows, cols, 128) ||
        !make_map_bf16(&tv, a.v, cols, rows, cols, 128) ||
        !make_map_bf16(&tkg, a.k, cols, rows, cols, 1) ||
        !make_map_bf16(&tvg, a.v, cols, rows, cols, 1))
        return cudaErrorInvalidValue;
    AttnParams p{};
    p.idx = a.idx;
    p.counts = a.counts;
    p.k_max = a.k_max;
    p.base = static_cast<const __nv_bfloat16*>(a.base);
    p.out = static_cast<__nv_bfloat16*>(a.out);
    p.scale = a.scale;
    p.row_max = a.row_max;
    p.exp_sum = a.exp_sum;
    p.prev_m = a.prev_m;
    p.prev_l = a.prev_l;
    p.colsum = a.colsum;
    p.layout = a.layout;
    p.heads = (int)a.heads;
    p.n = (int)a.n;
    p.chunk = (int)a.chunk;
    p.chunks = (int)(a.n / a.chunk);
    p.kp = static_cast<const __nv_bfloat16*>(a.k);
    p.vp = static_cast<const __nv_bfloat16*>(a.v);
    {
        // sparse K/V staging path: cp.async copy warps (default) or TMA gather4
        // (CSD_ATTN_GATHER=g4, for comparison)
        static const int cp = [] {
            const char* e = std::getenv("CSD_ATTN_GATHER");
            return (e && std::string(e) == "g4") ? 0 : 1;
        }();
        p.cp_async = cp;
    }
    p.trace = h_attn_trace;
    p.span = h_attn_span;
    p.cs_chunk = (a.colsum != nullptr && a.cs_chunk > 0 && a.cs_chunk != a.chunk) ? (int)a.cs_chunk : 0;
    p.cs_chunks = p.cs_chunk ? (int)(a.n / a.cs_chunk) : 0;
    if (p.cs_chunk) {  // items straddle colsum chunks: the two partial sums are atomically merged
        cudaError_t e = cudaMemsetAsync(a.colsum, 0, sizeof(float) * a.batch * a.heads * p.cs_chunks * a.n, s);
        if (e != cudaSuccess) return e;
    }
    p.items = (int)(a.batch * a.heads * p.chunks);
    p.qk_scale_log2 = kLog2e / std::sqrt((float)E);

    // ---- shared-memory layout (see AttnLayout)
    {
        auto al = [](uint32_t v) { return (v + 1023u) & ~1023u; };
        uint32_t off = 0;
        for (int t = 0; t < 2; ++t) {
            const int rows_t = t < NT ? (int)((std::min<int64_t>(128, a.chunk - 128 * t) + 63) / 64 * 64) : 0;
            p.q_rows[t] = rows_t;
            p.q_off[t] = off;
            p.q_strip[t] = (uint32_t)rows_t * 128u;
            off = al(off + L::kHalves * p.q_strip[t]);
        }
        const uint32_t xrows = (uint32_t)((a.chunk + 63) / 64 * 64);
        const uint32_t xbase = L::kHalves * xrows * 128u;
        // rings, row-half exchange, barriers (the dynamic smem window is 1 KB aligned: no
        // slack, the kernel traps otherwise)
        const uint32_t tail = 4 * L::kKV + L::kXchBytes + 256;
        const bool want = a.base != nullptr && a.colsum == nullptr && off + xbase + tail <= L::kMaxSmem;
        p.stage_base = want ? 1 : 0;
        p.x_strip = xrows * 128u;
        p.off_x = off;
        off = al(off + (want ? std::max(xbase, L::kCsBytes) : L::kCsBytes));
        p.off_k = off;
        p.off_v = off + 2 * L::kKV;
        p.off_xch = p.off_v + 2 * L::kKV;
        p.off_bar = p.off_xch + L::kXchBytes;
    }
    const uint32_t smem_bytes = p.off_bar + 256;
    if (smem_bytes > L::kMaxSmem) return cudaErrorNotSupported;
    auto kern = k_attn_tc<E, NT>;
    {
        cudaError_t err = ensure_smem_attr(kern, (int)L::kMaxSmem);  // per device
        if (err != cudaSuccess) return err;
    }
    const int sms = sm_count();
    // persistent: one CTA per SM (smem-limited), items strided over the grid
    const unsigned grid = (unsigned)std::min<int64_t>(p.items, sms);
    kern<<<grid, L::kThreads, smem_bytes, s>>>(tq, tk, tv, tkg, tvg, tb, to, p);
    return cudaGetLastError();
}

cudaError_t attn_tc(const AttnTcArgs& a, cudaStream_t s) {
    if (!attn_tc_supported(a.e, a.chunk)) return cudaErrorNotSupported;
    if (a.n % a.chunk) return cudaErrorInvalidValue;
    if (attn_sd_supported(a)) return attn_sd(a, s);
    if (attn_px_supported(a)) return attn_px(a, s);
    if (attn_cp_supported(a)) return attn_cp(a, s);
    if (attn_pp_supported(a)) return attn_pp(a, s);
    const bool two = a.chunk > 128;
    if (a.e == 128) return two ? launch_attn<128, 2>(a, s) : launch_attn<128, 1>(a, s);
    return two ? launch_attn<64, 2>(a, s) : launch_attn<64, 1>(a, s);
}

}  // namespace dev
}  // namespace csd

// Debug only (scripts/attn_trace.py): point the attention kernels' timeline buffer at a
// device array of kTraceCtas * kTraceSlots uint64 (nullptr disables tracing).
extern "C" int csd_debug_set_attn_trace(void* dev_buf) {
    uint64_t* p = static_cast<uint64_t*>(dev_buf);
    csd::dev::h_attn_trace = p;
    return 0;
}
// Debug only: per-CTA [start, end] globaltimer stamps (2 x grid uint64).
extern "C" int csd_debug_set_attn_span(void* dev_buf) {
    uint64_t* p = static_cast<uint64_t*>(dev_buf);
    csd::dev::h_attn_span = p;
    return 0;
}
