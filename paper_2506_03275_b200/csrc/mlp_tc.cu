// mlp_tc.cu — sparse-delta MLP on tcgen05 (CSD_MODE_PROD), mlp.cpp:120-182.
//
// Per token chunk z (c rows, index set S_z of `cnt` neurons):
//   up   (k_smlp_up)  : P = x_c W1[S]^T           M=c (NT x 128 tiles) N=128 neurons K=D
//                       epilogue: a = gelu(P + b1[S]); delta = a - A_cache[z, S, :];
//                       A_cache[z, S, :] = a  (chunk-major cache: each selected neuron's
//                       c activations are contiguous, so the read-modify-write coalesces);
//                       delta -> workspace [z][row][k_pad] bf16 (zeros past cnt)
//   down (k_smlp_down): M_cache[z rows, :] += delta W2[S]   M=c N=128 of D K=cnt
//                       (W2 rows gathered by TMA gather4 into an MN-major B tile; the
//                       epilogue is the O = O_cache + delta update, north_star item 5)
// Both kernels: warp 0 = TMA producer (x / delta tiles + gather4 of weight rows),
// warp 1 = single-thread tcgen05.mma issuer, warps 4.. = TMEM -> register epilogue.
// 4-stage smem ring (48 KB per stage), fp32 accumulators in TMEM.
#include <algorithm>

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "launch_util.h"
#include "tc_common.cuh"

namespace csd {
namespace dev {

using namespace csd::tc;

bool make_map_bf16(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows,
                   uint64_t pitch_elems, uint32_t box_rows);
bool make_map_2d(CUtensorMap* m, const void* base, int elem_bytes, uint64_t cols, uint64_t rows,
                 uint64_t pitch_elems, uint32_t box_cols, uint32_t box_rows, int swizzle_bytes);

// Debug timeline (scripts/mlp_trace.py): CTAs with blockIdx.y == 0 and blockIdx.x < 8
// record clock64() at fixed slots when the pointer is set.
// debug timeline buffer: host setting, passed in the kernel parameters (constant bank)
static uint64_t* h_mlp_trace = nullptr;
#define MLP_TRACE(slot)                                                                   \
    do {                                                                                  \
        uint64_t* tr_ = p.trace;                                                          \
        if (tr_ != nullptr && blockIdx.y == 0 && blockIdx.x < 8 && (slot) < 256)          \
            tr_[blockIdx.x * 256 + (slot)] = clock64();                                   \
    } while (0)

constexpr int kMlpStages = 4;  // 4 x 48 KB: one CTA per SM, deep enough to cover L2 latency
constexpr uint32_t kTile = 128 * 128;  // 128 rows x 64 bf16 (128 B) = 16 KB

template <int NT>
struct MlpLayout {
    static constexpr uint32_t kA = 0;                            // [stage][NT] 16 KB
    static constexpr uint32_t kB = kA + kMlpStages * NT * kTile; // [stage] 16 KB
    static constexpr uint32_t kBar = kB + kMlpStages * kTile;
    static constexpr uint32_t kBytes = kBar + 128 + 1024;  // barriers + staged ids / biases
    static constexpr uint32_t kSmemAlloc = kBytes + 1024;
    static constexpr uint32_t kThreads = 128 + 128 * NT;
    static constexpr uint32_t kTmemCols = NT * 128 <= 128 ? 128 : 256;
};

struct MlpParams {
    uint64_t* trace;  // debug timeline (null: off)
    const __nv_bfloat16* w1;  // gathered rows are staged with cp.async from these
    const __nv_bfloat16* w2;
    const int32_t* idx;
    const int32_t* counts;
    int k_max, k_pad;
    int tn_width;  // neurons per up-projection tile (multiple of 16, <= kUpMaxTN)
    int nz;        // chunks (batch x C)
    const float* b1;
    __nv_bfloat16* act_cm;
    __nv_bfloat16* delta;
    float* out_cache;
    const __nv_bfloat16* x_mid;  // optional fused residual: x_out = x_mid + out_cache
    __nv_bfloat16* x_out;
    int n, chunk, chunks, f, d;
};

// x_out[row, c0..c0+31] = bf16(x_mid + m) for 32 fp32 values m
__device__ __forceinline__ void residual32(const MlpParams& p, int64_t row, int col0,
                                           const float* m) {
    const uint4* xm = reinterpret_cast<const uint4*>(p.x_mid + row * p.d + col0);
    uint4* xo = reinterpret_cast<uint4*>(p.x_out + row * p.d + col0);
    uint4 xv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) xv[q] = xm[q];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint4 v = xv[q];
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
        uint4 o;
        uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float2 f = __bfloat1622float2(h[u]);
            ow[u] = pack_bf16x2(f.x + m[q * 8 + 2 * u], f.y + m[q * 8 + 2 * u + 1]);
        }
        xo[q] = o;
    }
}

template <int NT>
__device__ __forceinline__ void mlp_setup(uint8_t* smem, uint64_t*& full, uint64_t*& empty,
                                          uint64_t*& done, uint32_t& tmem, uint32_t full_count) {
    using L = MlpLayout<NT>;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
    full = bars;
    empty = bars + kMlpStages;
    done = bars + 2 * kMlpStages;
    uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 2 * kMlpStages + 1);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kMlpStages; ++s) {
            mbar_init(full + s, full_count);
            mbar_init(empty + s, 1);
        }
        mbar_init(done, 1);
        fence_barrier_init();
    }
    if ((threadIdx.x >> 5) == 1) tmem_alloc<L::kTmemCols>(slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    tmem = *slot;
}

// ------------------------------------------------------------------ up projection
// Tile = (chunk z, neuron tile tn of TN = p.tn_width neurons; TN is picked on the host so
// that all tiles run in ONE wave on 148 SMs, e.g. FLUX 860 -> 6 x 144).  MMA: M = chunk
// rows (NT x 128), N = TN, K = D.  Stage = x tile (TMA) + TN gathered W1 k-slices (cp.async).
constexpr int kUpMaxTN = 240;  // TMEM: NT x 240 <= 512 columns; see smlp_geometry for the smem cap
template <int NT>
struct UpLayout {
    static constexpr uint32_t kStageMax = NT * kTile + kUpMaxTN * 128;
    static constexpr uint32_t kThreads = 128 + 128 * NT;
    static constexpr uint32_t kBarBytes = 128 + 1024 + 1024;  // barriers, ids, biases
    static constexpr uint32_t kMaxSmem = 227 * 1024;
    static constexpr uint32_t kTmemCols = NT * kUpMaxTN <= 256 ? 256 : 512;
    __host__ __device__ static constexpr uint32_t stage_bytes(int tn) {
        return NT * kTile + (uint32_t)tn * 128u;
    }
    __host__ __device__ static constexpr int stages(int tn) {
        return (4 * stage_bytes(tn) + kBarBytes + 1024 <= kMaxSmem) ? 4 : 3;
    }
    __host__ __device__ static constexpr uint32_t alloc(int tn) {
        return stages(tn) * stage_bytes(tn) + kBarBytes + 1024;
    }
};

template <int NT>
__global__ void __launch_bounds__(UpLayout<NT>::kThreads, 1)
k_smlp_up(const __grid_constant__ CUtensorMap tm_x, const MlpParams p) {
    using L = UpLayout<NT>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int z = blockIdx.y, tn = blockIdx.x, TN = p.tn_width;
    pdl_wait();  // the counts / indices come from the previous kernel (top-k)
    if (threadIdx.x == 0) pdl_trigger();
    const int cnt = p.counts[z];
    const int n0 = tn * TN;  // first neuron slot of this tile
    const int b = z / p.chunks, c = z % p.chunks;
    const int x_row0 = b * p.n + c * p.chunk;
    const int kblocks = p.d / 64;
    const int nst = L::stages(TN);
    const uint32_t sbytes = L::stage_bytes(TN);
    const int32_t* ids = p.idx + (int64_t)z * p.k_max;
    const int nval = max(0, min(TN, cnt - n0));  // live neurons in this tile
    // delta rows of this chunk: [z * chunk + r][k_pad]
    __nv_bfloat16* drow0 = p.delta + (int64_t)z * p.chunk * p.k_pad;

    uint8_t* barp = smem + nst * sbytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(barp);
    uint64_t* empty = full + 4;
    uint64_t* done = full + 8;
    uint32_t* slot = reinterpret_cast<uint32_t*>(full + 9);
    int32_t* s_ids = reinterpret_cast<int32_t*>(barp + 128);
    float* s_b1 = reinterpret_cast<float*>(barp + 128 + 1024);
    constexpr int kCopyThreads = L::kThreads - 32;
    if (nval == 0) {
        // no live neuron: this tile's delta columns are zero (the down GEMM reads them)
        for (int idx = threadIdx.x; idx < p.chunk * (TN / 8); idx += blockDim.x) {
            const int r = idx / (TN / 8), pc = idx - r * (TN / 8);
            *reinterpret_cast<uint4*>(drow0 + (int64_t)r * p.k_pad + n0 + pc * 8) = make_uint4(0, 0, 0, 0);
        }
        return;
    }
    if (threadIdx.x == 0) {
        MLP_TRACE(0);
        for (int s = 0; s < nst; ++s) {
            // the x-tile expect_tx arrival + one cp.async-tracking arrival per copy thread
            mbar_init(full + s, 1 + kCopyThreads);
            mbar_init(empty + s, 1);
        }
        mbar_init(done, 1);
        fence_barrier_init();
    }
    for (int i = threadIdx.x; i < TN; i += blockDim.x) {
        const int nn = n0 + i;
        const int neuron = ids[nn < cnt ? nn : cnt - 1];  // pad: a valid row (column unused)
        s_ids[i] = neuron;
        s_b1[i] = p.b1[neuron];
    }
    if (warp == 1) tmem_alloc<L::kTmemCols>(slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (threadIdx.x == 0) MLP_TRACE(1);

    if (warp != 1) {
        // Producers = every warp but the MMA warp (the epilogue warps are idle until the
        // accumulator is final).  Warp 0 lane 0 issues the x tiles by TMA; the TN gathered
        // W1 rows of each stage are staged with cp.async, 16-byte pieces, the 8 pieces of a
        // row's 128-byte k-slice on consecutive threads (scripts/gather_bench2.cu: ~2.6x
        // TMA tile::gather4's per-SM rate).  A thread's rows are fixed for the whole K loop.
        const int ct = threadIdx.x < 32 ? threadIdx.x : threadIdx.x - 32;
        constexpr int kPer = (kUpMaxTN * 8 + kCopyThreads - 1) / kCopyThreads;
        const char* src[kPer];
        uint32_t dso[kPer];
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const int idx = ct + i * kCopyThreads;
            const int row = idx >> 3, c8 = idx & 7;
            const bool ok = row < TN;
            src[i] = reinterpret_cast<const char*>(p.w1 + (int64_t)s_ids[ok ? row : 0] * p.d) + c8 * 16;
            dso[i] = ok ? (uint32_t)(NT * kTile + row * 128 + ((c8 ^ (row & 7)) << 4)) : 0xffffffffu;
        }
        if (warp == 0 && lane == 0) tma_prefetch_desc(&tm_x);
        const uint32_t s0 = smem_u32(smem);
        for (int kb = 0; kb < kblocks; ++kb) {
            const int s = kb % nst;
            if (kb == nst && warp == 4) {
                // warm L2 with this tile's activation-cache rows (the epilogue's input)
                const __nv_bfloat16* cache_z = p.act_cm + (int64_t)z * p.f * p.chunk;
                for (int n = lane; n < nval; n += 32)
                    bulk_prefetch_l2(cache_z + (int64_t)s_ids[n] * p.chunk, (uint32_t)p.chunk * 2u);
            }
            if (kb >= nst) mbar_wait(empty + s, ((kb / nst) - 1) & 1);
            if (warp == 0 && lane == 0) {
                MLP_TRACE(2 + kb);
                // only the chunk's rows (64-row boxes); the MMA's rows past the chunk read
                // stale smem -- dead accumulator rows that are never stored
                const int nbox = (p.chunk + 63) >> 6;
                mbar_arrive_expect_tx(full + s, (uint32_t)nbox * 8192u);
                for (int bx = 0; bx < nbox; ++bx)
                    tma_load_2d(&tm_x, full + s, smem + s * sbytes + (bx >> 1) * kTile + (bx & 1) * 8192,
                                kb * 64, x_row0 + bx * 64);
            }
#pragma unroll
            for (int i = 0; i < kPer; ++i)
                if (dso[i] != 0xffffffffu)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s0 + s * sbytes + dso[i]),
                                 "l"(src[i] + kb * 128) : "memory");
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full + s)) : "memory");
        }
    }
    if (warp == 1) {
        if (lane == 0) {
            const uint32_t id = idesc_bf16(128, (uint32_t)TN, false, false);
            const uint32_t s0 = smem_u32(smem);
            for (int kb = 0; kb < kblocks; ++kb) {
                const int s = kb % nst;
                mbar_wait(full + s, (kb / nst) & 1);
                fence_proxy_async_smem();  // cp.async (generic proxy) data -> tcgen05 reads
                tc_fence_after();
                MLP_TRACE(64 + kb);
                const uint32_t sa = s0 + s * sbytes, sb = sa + NT * kTile;
                for (int t = 0; t < NT; ++t) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_bf16(tmem + t * kUpMaxTN, desc_kmajor_sw128(sa + t * kTile + kk * 32),
                                 desc_kmajor_sw128(sb + kk * 32), id, (kb > 0 || kk > 0) ? 1u : 0u);
                }
                mma_commit(empty + s);
            }
            mma_commit(done);
        }
    } else if (warp >= 4) {
        // Staged epilogue in the (now idle) stage ring:
        //   act tile   [TN neurons][chunk rows] bf16: a selected neuron's chunk-major cache row
        //              is contiguous (chunk x 2 B): coalesced 16-byte cp.async in / stores out;
        //   delta tile [chunk rows][TN] bf16, row pitch TN * 2 + 16 B (bank-conflict free),
        //              written out row-contiguously.
        // Thread = chunk row: a warp's smem accesses hit consecutive rows.
        const int sw = warp - 4, t = sw >> 2, quad = warp & 3;
        const int r = t * 128 + quad * 32 + lane;  // row within the chunk
        const bool row_ok = r < p.chunk;
        const int ept = threadIdx.x - 128;
        const uint32_t row_bytes = (uint32_t)p.chunk * 2u;
        const int pieces = (int)(row_bytes / 16u);
        const uint32_t dp = (uint32_t)TN * 2u + 16u;
        uint8_t* stg_act = smem;
        uint8_t* stg_dl = smem + (((uint32_t)TN * row_bytes + 1023u) & ~1023u);
        mbar_wait(done, 0);  // all MMAs done: the ring is free
        tc_fence_after();
        if (sw == 0 && lane == 0) MLP_TRACE(128);
        {
            const char* cache_z = reinterpret_cast<const char*>(p.act_cm + (int64_t)z * p.f * p.chunk);
            for (int idx = ept; idx < nval * pieces; idx += 128 * NT) {
                const int n = idx / pieces, pc = idx - n * pieces;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(stg_act + n * row_bytes + pc * 16)),
                             "l"(cache_z + (int64_t)s_ids[n] * row_bytes + pc * 16) : "memory");
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        }
        named_bar_sync(1, 128 * NT);  // the whole act tile has landed
        if (sw == 0 && lane == 0) MLP_TRACE(130);
        const uint32_t tacc = tmem + ((uint32_t)(quad * 32) << 16) + t * kUpMaxTN;
#pragma unroll 1
        for (int g = 0; g < TN / 16; ++g) {
            uint32_t acc[16];
            tmem_ld16(tacc + g * 16, acc);
            tmem_ld_wait();
            if (!row_ok) continue;
            uint32_t pk[8];
            __nv_bfloat16* ap0 = reinterpret_cast<__nv_bfloat16*>(stg_act + g * 16 * row_bytes) + r;
            const int nv = nval - g * 16;  // live neurons in this group (uniform)
            if (nv >= 16) {  // branch-free: the 16 chains interleave
                float an[16], ol[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) ol[i] = __bfloat162float(ap0[i * (row_bytes / 2)]);
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    an[i] = __bfloat162float(__float2bfloat16_rn(
                        gelu_tanh_approx(__uint_as_float(acc[i]) + s_b1[g * 16 + i])));
#pragma unroll
                for (int i = 0; i < 16; ++i) ap0[i * (row_bytes / 2)] = __float2bfloat16_rn(an[i]);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    pk[i] = pack_bf16x2(an[2 * i] - ol[2 * i], an[2 * i + 1] - ol[2 * i + 1]);
            } else {
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                    float d2[2];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        __nv_bfloat16* ap = ap0 + (i + u) * (row_bytes / 2);
                        const float a = gelu_tanh_approx(__uint_as_float(acc[i + u]) + s_b1[g * 16 + i + u]);
                        const __nv_bfloat16 a16 = __float2bfloat16_rn(a);
                        d2[u] = 0.f;
                        if (i + u < nv) {
                            d2[u] = __bfloat162float(a16) - __bfloat162float(*ap);
                            *ap = a16;
                        }
                    }
                    pk[i / 2] = pack_bf16x2(d2[0], d2[1]);
                }
            }
            uint4* dd = reinterpret_cast<uint4*>(stg_dl + r * dp + g * 32);
            dd[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            dd[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
        named_bar_sync(1, 128 * NT);
        if (sw == 0 && lane == 0) MLP_TRACE(131);
        {   // act tile out and delta tile out: coalesced 16-byte stores
            char* cache_z = reinterpret_cast<char*>(p.act_cm + (int64_t)z * p.f * p.chunk);
            for (int idx = ept; idx < nval * pieces; idx += 128 * NT) {
                const int n = idx / pieces, pc = idx - n * pieces;
                *reinterpret_cast<uint4*>(cache_z + (int64_t)s_ids[n] * row_bytes + pc * 16) =
                    *reinterpret_cast<const uint4*>(stg_act + n * row_bytes + pc * 16);
            }
            const int dpc = TN / 8;  // 16-byte pieces per delta row of this tile
            for (int idx = ept; idx < p.chunk * dpc; idx += 128 * NT) {
                const int rr = idx / dpc, pc = idx - rr * dpc;
                *reinterpret_cast<uint4*>(drow0 + (int64_t)rr * p.k_pad + n0 + pc * 8) =
                    *reinterpret_cast<const uint4*>(stg_dl + rr * dp + pc * 16);
            }
            // the last tile also zeroes the padding columns [n0 + TN, k_pad) the down GEMM reads
            if (n0 + TN < p.k_pad && (tn + 1) * TN >= cnt) {
                const int zc = (p.k_pad - n0 - TN) / 8;
                for (int idx = ept; idx < p.chunk * zc; idx += 128 * NT) {
                    const int rr = idx / zc, pc = idx - rr * zc;
                    *reinterpret_cast<uint4*>(drow0 + (int64_t)rr * p.k_pad + n0 + TN + pc * 8) =
                        make_uint4(0, 0, 0, 0);
                }
            }
        }
    }
    if (threadIdx.x == 128) MLP_TRACE(129);
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<L::kTmemCols>(tmem);
    }
}

// ------------------------------------------------------------------ down projection
// Persistent: item = (chunk z, 128-column D tile td), items strided over min(items, SMs)
// CTAs.  Per item: M_cache[z rows, td cols] += delta[z rows, :cnt] W2[S][:, td cols]
// (M = chunk rows as NT x 128, N = 128, K = cnt in 64-neuron k-blocks), then the residual
// x_out = x_mid + M_cache (north_star item 5: the cache update fused into the epilogue).
// The TMEM accumulator is double-buffered so an item's epilogue overlaps the next item's
// K loop.  Stage = delta tile (TMA) + 64 gathered W2 rows x 128 columns (cp.async, MN-major).
//
// Epilogue through TMA: an item's 128 columns are four 32-column slices; each slice's
// M_cache rows (fp32, 128 B per row, 128B swizzle) and x_mid rows (bf16, 64 B, 64B swizzle)
// are TMA-loaded into one of two slice buffers ahead of use (the loads do not depend on the
// accumulator, so they run ahead of the K loop), updated in place by thread = chunk row
// (the swizzles keep a warp's 16-byte accesses conflict-free), and TMA-stored back.  The
// read-modify-write is then bound by the TMA engine's bytes in flight, not by the
// per-thread register budget of a load -> use -> store loop.
template <int NT>
struct DnLayout {
    static constexpr uint32_t kStage = NT * kTile + kTile;  // A (rows x 64 k) + B (64 k x 128)
    // warps 0 (TMA + copy), 1 (MMA), 2-3 (copy), 4 .. 4 + 4 NT - 1 (epilogue), then 4 more
    // copy warps: the W2 row gather (cp.async, LSU rate per issuing warp) is the K loop's limiter
    static constexpr uint32_t kThreads = 256 + 128 * NT;
    static constexpr uint32_t kTmemCols = 2 * NT * 128 <= 256 ? 256 : 512;
    static constexpr uint32_t kMaxSmem = 227 * 1024;
    static constexpr uint32_t kBarBytes = 256;
    __host__ __device__ static constexpr uint32_t ebuf_m(int chunk) { return ((uint32_t)chunk * 128u + 1023u) & ~1023u; }
    __host__ __device__ static constexpr uint32_t ebuf_x(int chunk) { return ((uint32_t)chunk * 64u + 1023u) & ~1023u; }
    __host__ __device__ static constexpr uint32_t ebytes(int chunk) { return 2u * (ebuf_m(chunk) + ebuf_x(chunk)); }
    __host__ __device__ static constexpr int stages(int chunk) {
        return (4 * kStage + ebytes(chunk) + kBarBytes + 1024 <= kMaxSmem)   ? 4
               : (3 * kStage + ebytes(chunk) + kBarBytes + 1024 <= kMaxSmem) ? 3
                                                                             : 2;
    }
    __host__ __device__ static constexpr uint32_t alloc(int chunk) {
        return stages(chunk) * kStage + ebytes(chunk) + kBarBytes + 1024;
    }
};

template <int NT>
__global__ void __launch_bounds__(DnLayout<NT>::kThreads, 1)
k_smlp_down(const __grid_constant__ CUtensorMap tm_delta, const __grid_constant__ CUtensorMap tm_mc,
            const __grid_constant__ CUtensorMap tm_xm, const __grid_constant__ CUtensorMap tm_xo,
            const MlpParams p) {
    using L = DnLayout<NT>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntd = p.d / 128;
    const int items = p.nz * ntd;
    const int nst = L::stages(p.chunk);
    uint8_t* ebase = smem + nst * L::kStage;  // [2] M slices, then [2] x slices
    uint64_t* bars = reinterpret_cast<uint64_t*>(ebase + L::ebytes(p.chunk));
    uint64_t* full = bars;           // [4]
    uint64_t* empty = bars + 4;      // [4]
    uint64_t* tfull = bars + 8;      // [2] accumulator buffer final
    uint64_t* tempty = tfull + 2;    // [2] accumulator buffer drained
    uint64_t* efull = tempty + 2;    // [2] epilogue slice buffer loaded
    uint32_t* slot = reinterpret_cast<uint32_t*>(efull + 2);
    constexpr int kCopyThreads = 224;         // warps 0, 2, 3 and the 4 trailing warps
    constexpr int kXtra = 4 + 4 * NT;         // first trailing copy warp
    if (threadIdx.x == 0) {
        MLP_TRACE(200);
        for (int s = 0; s < nst; ++s) {
            mbar_init(full + s, 1 + kCopyThreads);
            mbar_init(empty + s, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(tfull + i, 1);
            mbar_init(tempty + i, 128 * NT);
            mbar_init(efull + i, 1);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<L::kTmemCols>(slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    pdl_wait();
    if (threadIdx.x == 0) pdl_trigger();
    auto kblocks_of = [&](int item) { return (p.counts[item / ntd] + 63) / 64; };

    if (warp == 0 || warp == 2 || warp == 3 || warp >= kXtra) {
        // producers: warp 0 lane 0 the delta tiles (TMA); all 224 threads the W2 k-slices,
        // one row's 16 pieces (2 strips x 8) on consecutive threads
        if constexpr (NT == 2) regs_dec<72>();  // 512 threads: the epilogue gets the registers
        const int ct = warp == 0 ? lane : warp < 4 ? (warp - 1) * 32 + lane : 96 + (warp - kXtra) * 32 + lane;
        constexpr int kPer = (64 * 16 + kCopyThreads - 1) / kCopyThreads;
        if (warp == 0 && lane == 0) tma_prefetch_desc(&tm_delta);
        const uint32_t s0 = smem_u32(smem);
        uint32_t gk = 0;  // global k-block counter (ring position)
        for (int item = blockIdx.x; item < items; item += gridDim.x) {
            const int z = item / ntd, td = item - z * ntd;
            const int cnt = p.counts[z];
            const int kbs = (cnt + 63) / 64;
            const int32_t* ids = p.idx + (int64_t)z * p.k_max;
            for (int kb = 0; kb < kbs; ++kb, ++gk) {
                const int s = gk % nst;
                int nid[kPer];
#pragma unroll
                for (int i = 0; i < kPer; ++i) {
                    const int idx = ct + i * kCopyThreads;
                    int nn = kb * 64 + ((idx >> 4) & 63);
                    nid[i] = __ldg(ids + (nn < cnt ? nn : cnt - 1));  // pad: a valid row (delta = 0)
                }
                if (gk >= (uint32_t)nst) mbar_wait(empty + s, ((gk / nst) - 1) & 1);
                if (warp == 0 && lane == 0) {
                    const int nbox = (p.chunk + 63) >> 6;  // only the chunk's rows
                    mbar_arrive_expect_tx(full + s, (uint32_t)nbox * 8192u);
                    for (int bx = 0; bx < nbox; ++bx)
                        tma_load_2d(&tm_delta, full + s, smem + s * L::kStage + (bx >> 1) * kTile + (bx & 1) * 8192,
                                    kb * 64, z * p.chunk + bx * 64);
                }
#pragma unroll
                for (int i = 0; i < kPer; ++i) {
                    const int idx = ct + i * kCopyThreads;
                    if (idx < 64 * 16) {
                        const int row = idx >> 4, piece = idx & 15;
                        const uint32_t d = s0 + s * L::kStage + NT * kTile + (piece >> 3) * 8192 + row * 128 +
                                           (((piece & 7) ^ (row & 7)) << 4);
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d),
                                     "l"(p.w2 + (int64_t)nid[i] * p.d + td * 128 + piece * 8) : "memory");
                    }
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full + s)) : "memory");
            }
        }
    } else if (warp == 1) {
        if constexpr (NT == 2) regs_dec<72>();
        if (lane == 0) {
            constexpr uint32_t id = idesc_bf16(128, 128, false, true);
            const uint32_t s0 = smem_u32(smem);
            uint32_t gk = 0, li = 0;
            for (int item = blockIdx.x; item < items; item += gridDim.x, ++li) {
                const int kbs = kblocks_of(item);
                const uint32_t ab = li & 1;
                if (li >= 2) mbar_wait(tempty + ab, ((li >> 1) - 1) & 1);  // buffer drained
                tc_fence_after();
                const uint32_t acc = tmem + ab * (NT * 128);
                if (kbs == 0) {  // nothing to accumulate: the epilogue adds zero
                    mma_commit(tfull + ab);
                    continue;
                }
                for (int kb = 0; kb < kbs; ++kb, ++gk) {
                    const int s = gk % nst;
                    mbar_wait(full + s, (gk / nst) & 1);
                    fence_proxy_async_smem();  // cp.async (generic proxy) data -> tcgen05 reads
                    tc_fence_after();
                    if (kb == 0 && li < 8) MLP_TRACE(202 + 2 * li);
                    const uint32_t sa = s0 + s * L::kStage, sb = sa + NT * kTile;
                    for (int t = 0; t < NT; ++t) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_bf16(acc + t * 128, desc_kmajor_sw128(sa + t * kTile + kk * 32),
                                     desc_mnmajor_sw128(sb + kk * 2048, 8192), id,
                                     (kb > 0 || kk > 0) ? 1u : 0u);
                    }
                    mma_commit(empty + s);
                }
                mma_commit(tfull + ab);
                if (li < 8) MLP_TRACE(203 + 2 * li);
            }
        }
    } else {
        // setmaxnreg.inc draws only on registers this CTA's decs released (8 warps x 56 at
        // 128 -> 72 fund exactly 8 warps x 56 at 128 -> 184); asking for more deadlocks
        if constexpr (NT == 2) regs_inc<184>();
        const int sw = warp - 4, t = sw >> 2, quad = warp & 3;
        const int r = t * 128 + quad * 32 + lane;  // chunk row (TMEM lane)
        const bool row_ok = r < p.chunk;
        const bool lead = sw == 0 && lane == 0;  // issues the slice loads and stores
        const bool has_x = p.x_out != nullptr;
        const uint32_t em = L::ebuf_m(p.chunk), ex = L::ebuf_x(p.chunk);
        const uint32_t tx_bytes = (uint32_t)p.chunk * (has_x ? 192u : 128u);
        const int my_items = (items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
        const int nslices = my_items * 4;
        auto slice_rc = [&](int sl, int& col, int& row0) {
            const int item = blockIdx.x + (sl >> 2) * gridDim.x;
            const int z = item / ntd, td = item - z * ntd;
            const int b = z / p.chunks, c = z - b * p.chunks;
            col = td * 128 + (sl & 3) * 32;
            row0 = b * p.n + c * p.chunk;
        };
        auto issue = [&](int sl) {  // lead only: load slice sl into buffer sl & 1
            if (sl >= nslices) return;
            int col, row0;
            slice_rc(sl, col, row0);
            const int bi = sl & 1;
            mbar_arrive_expect_tx(efull + bi, tx_bytes);
            tma_load_2d(&tm_mc, efull + bi, ebase + bi * em, col, row0);
            if (has_x) tma_load_2d(&tm_xm, efull + bi, ebase + 2 * em + bi * ex, col, row0);
        };
        if (lead) {
            tma_prefetch_desc(&tm_mc);
            if (has_x) { tma_prefetch_desc(&tm_xm); tma_prefetch_desc(&tm_xo); }
            issue(0);
            issue(1);
        }
        uint32_t li = 0;
        int sl = 0;
        for (int item = blockIdx.x; item < items; item += gridDim.x, ++li) {
            const int z = item / ntd;
            const bool has_acc = p.counts[z] > 0;
            const uint32_t ab = li & 1;
            mbar_wait(tfull + ab, (li >> 1) & 1);
            tc_fence_after();
            if (sw == 0 && lane == 0 && li < 8) MLP_TRACE(230 + 2 * li);
            const uint32_t tacc = tmem + ab * (NT * 128) + ((uint32_t)(quad * 32) << 16) + t * 128;
            for (int oc = 0; oc < 4; ++oc, ++sl) {
                uint32_t v[32];
                if (has_acc) {
                    tmem_ld32(tacc + oc * 32, v);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = 0u;
                }
                if (oc == 3) {  // TMEM reads of this buffer done: let the next-but-one item in
                    tc_fence_before();
                    mbar_arrive(tempty + ab);
                }
                const int bi = sl & 1;
                mbar_wait(efull + bi, (sl >> 1) & 1);
                if (row_ok) {
                    // M row: 8 x 16 B at chunk position q ^ (r & 7) (128B swizzle)
                    float* mrow = reinterpret_cast<float*>(ebase + bi * em + r * 128);
                    float mv[32];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        float4* pm = reinterpret_cast<float4*>(mrow + ((q ^ (r & 7)) << 2));
                        float4 a = *pm;
                        a.x += __uint_as_float(v[4 * q]);
                        a.y += __uint_as_float(v[4 * q + 1]);
                        a.z += __uint_as_float(v[4 * q + 2]);
                        a.w += __uint_as_float(v[4 * q + 3]);
                        *pm = a;
                        mv[4 * q] = a.x;
                        mv[4 * q + 1] = a.y;
                        mv[4 * q + 2] = a.z;
                        mv[4 * q + 3] = a.w;
                    }
                    if (has_x) {
                        // x row: 4 x 16 B at chunk position q ^ ((r >> 1) & 3) (64B swizzle)
                        uint4* xrow = reinterpret_cast<uint4*>(ebase + 2 * em + bi * ex + r * 64);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            uint4* px = xrow + (q ^ ((r >> 1) & 3));
                            uint4 xv = *px;
                            uint32_t* w = reinterpret_cast<uint32_t*>(&xv);
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[u]));
                                w[u] = pack_bf16x2(f.x + mv[8 * q + 2 * u], f.y + mv[8 * q + 2 * u + 1]);
                            }
                            *px = xv;
                        }
                    }
                }
                fence_proxy_async_smem();  // generic-proxy smem writes -> the TMA store
                named_bar_sync(1, 128 * NT);
                if (lead) {
                    int col, row0;
                    slice_rc(sl, col, row0);
                    tma_store_2d(&tm_mc, ebase + bi * em, col, row0);
                    if (has_x) tma_store_2d(&tm_xo, ebase + 2 * em + bi * ex, col, row0);
                    bulk_commit();
                    bulk_wait_read0();  // the store has read buffer bi: reuse it
                    issue(sl + 2);
                }
            }
            if (sw == 0 && lane == 0 && li < 8) MLP_TRACE(231 + 2 * li);
        }
        if (lead) bulk_wait0();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<L::kTmemCols>(tmem);
    }
}

bool mlp_tc_supported(int64_t d, int64_t chunk) {
    // chunk % 8: a neuron's chunk-major cache row (chunk x 2 B) moves by 16-byte bulk copies
    return d % 128 == 0 && chunk >= 8 && chunk <= 256 && chunk % 8 == 0;
}

void smlp_geometry(int64_t k_max, int64_t nz, int64_t chunk, int* tn_width, int* ntiles, int64_t* k_pad);

template <int NT>
static cudaError_t launch_smlp(const void* x, const void* w1, const float* b1, const void* w2,
                               const int32_t* idx, const int32_t* counts, int64_t k_max,
                               int64_t chunk, int64_t batch, int64_t n, int64_t d, int64_t f,
                               void* act_cm, float* out_cache, void* delta_ws, int64_t k_pad,
                               cudaStream_t s, const void* x_mid, void* x_out) {
    using L = MlpLayout<NT>;
    using LU = UpLayout<NT>;
    const int64_t nc = n / chunk;
    int tn_width = 0, ntiles = 0;
    smlp_geometry(k_max, batch * nc, chunk, &tn_width, &ntiles, nullptr);
    CUtensorMap tx, tdl, tmc, txm, txo;
    const uint64_t rows_all = (uint64_t)(batch * n);
    if (!make_map_bf16(&tx, x, d, batch * n, d, 64) ||
        !make_map_bf16(&tdl, delta_ws, k_pad, batch * nc * chunk, k_pad, 64) ||
        !make_map_2d(&tmc, out_cache, 4, d, rows_all, d, 32, (uint32_t)chunk, 128) ||
        !make_map_2d(&txm, x_mid != nullptr ? x_mid : x, 2, d, rows_all, d, 32, (uint32_t)chunk, 64) ||
        !make_map_2d(&txo, x_out != nullptr ? x_out : x, 2, d, rows_all, d, 32, (uint32_t)chunk, 64))
        return cudaErrorInvalidValue;
    MlpParams p{};
    p.trace = h_mlp_trace;
    p.w1 = (const __nv_bfloat16*)w1;
    p.w2 = (const __nv_bfloat16*)w2;
    p.idx = idx;
    p.counts = counts;
    p.k_max = (int)k_max;
    p.k_pad = (int)k_pad;
    p.tn_width = tn_width;
    p.b1 = b1;
    p.act_cm = (__nv_bfloat16*)act_cm;
    p.delta = (__nv_bfloat16*)delta_ws;
    p.out_cache = out_cache;
    p.x_mid = (const __nv_bfloat16*)x_mid;
    p.x_out = (__nv_bfloat16*)x_out;
    p.n = (int)n;
    p.chunk = (int)chunk;
    p.chunks = (int)nc;
    p.f = (int)f;
    p.d = (int)d;
    p.nz = (int)(batch * nc);
    {
        cudaError_t e = ensure_smem_attr(k_smlp_up<NT>, (int)LU::kMaxSmem);
        if (e == cudaSuccess) e = ensure_smem_attr(k_smlp_down<NT>, (int)DnLayout<NT>::kMaxSmem);
        if (e != cudaSuccess) return e;
    }
    dim3 g1((unsigned)ntiles, (unsigned)(batch * nc));
    cudaError_t e = launch_ex(k_smlp_up<NT>, g1, dim3(LU::kThreads), LU::alloc(tn_width), s, 1, tx, p);
    if (e != cudaSuccess) return e;
    const int sms = sm_count();
    const int64_t items = batch * nc * (d / 128);
    return launch_ex(k_smlp_down<NT>, dim3((unsigned)std::min<int64_t>(items, sms)),
                     dim3(DnLayout<NT>::kThreads), DnLayout<NT>::alloc((int)chunk), s, 1, tdl, tmc,
                     txm, txo, p);
}

// Up-projection tiling: as many neuron tiles per chunk as fit ONE wave over the SMs
// (FLUX: 24 chunks -> 6 tiles of 144 for k = 860), width a multiple of 16 in [64, 192].
// The delta workspace is [B*C*chunk rows][k_pad] bf16, k_pad = round_up(tiles * width, 64)
// (the down GEMM's 64-neuron k-blocks read up to round_up(count, 64) columns).
void smlp_geometry(int64_t k_max, int64_t nz, int64_t chunk, int* tn_width, int* ntiles, int64_t* k_pad) {
    const int sms = sm_count();
    const int64_t km = std::max<int64_t>(k_max, 1);
    const int64_t fit = std::max<int64_t>(1, sms / std::max<int64_t>(nz, 1));
    // widest tile: its epilogue stages the activation tile [TN][chunk] and the delta tile
    // [chunk][TN + 8] (bf16) in the idle stage ring, which must hold them
    auto staging_fits = [&](int64_t w) {
        const int nt = chunk > 128 ? 2 : 1;
        const int64_t stage = nt * (int64_t)kTile + w * 128;
        const int64_t ring = (4 * stage + 128 + 2048 + 1024 <= 227 * 1024 ? 4 : 3) * stage;
        const int64_t need = ((w * chunk * 2 + 1023) / 1024) * 1024 + chunk * (w * 2 + 16);
        return need <= ring;
    };
    int64_t wmax = 192;  // the round-1 envelope: always fits
    for (int64_t w = kUpMaxTN; w > 192; w -= 16)
        if (staging_fits(w)) {
            wmax = w;
            break;
        }
    int64_t w = (km + fit - 1) / fit;
    w = (w + 15) / 16 * 16;
    // one wave at <= wmax neurons per tile; past that the tiles run in several waves anyway
    // and the narrower 192 measured faster (FLUX 85 %: 186 vs 200 us)
    w = std::max<int64_t>(w, 64);
    if (w > wmax) w = 192;
    const int64_t t = (km + w - 1) / w;
    if (tn_width) *tn_width = (int)w;
    if (ntiles) *ntiles = (int)t;
    if (k_pad) *k_pad = (t * w + 63) / 64 * 64;
}

int64_t prod_smlp_delta_cols(int64_t k_max, int64_t nz, int64_t chunk) {
    int64_t k_pad = 0;
    smlp_geometry(k_max, nz, chunk, nullptr, nullptr, &k_pad);
    return k_pad;
}

cudaError_t prod_sparse_delta_mlp_tc(const void* x, const void* w1, const float* b1,
                                     const void* w2, const int32_t* idx, const int32_t* counts,
                                     int64_t k_max, int64_t chunk, int64_t batch, int64_t n,
                                     int64_t d, int64_t f, void* act_cm, float* out_cache,
                                     void* delta_ws, cudaStream_t s, const void* x_mid,
                                     void* x_out) {
    if (!mlp_tc_supported(d, chunk)) return cudaErrorNotSupported;
    if (k_max == 0) return cudaSuccess;
    int64_t k_pad = 0;
    smlp_geometry(k_max, batch * (n / chunk), chunk, nullptr, nullptr, &k_pad);
    if (chunk > 128)
        return launch_smlp<2>(x, w1, b1, w2, idx, counts, k_max, chunk, batch, n, d, f, act_cm,
                              out_cache, delta_ws, k_pad, s, x_mid, x_out);
    return launch_smlp<1>(x, w1, b1, w2, idx, counts, k_max, chunk, batch, n, d, f, act_cm,
                          out_cache, delta_ws, k_pad, s, x_mid, x_out);
}

}  // namespace dev
}  // namespace csd

// Debug only (scripts/mlp_trace.py): timeline buffer of 8 x 256 uint64 for k_smlp_up.
extern "C" int csd_debug_set_mlp_trace(void* dev_buf) {
    uint64_t* p = static_cast<uint64_t*>(dev_buf);
    csd::dev::h_mlp_trace = p;
    return 0;
}
