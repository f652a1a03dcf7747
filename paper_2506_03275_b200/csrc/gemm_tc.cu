// gemm_tc.cu — persistent tcgen05 GEMM with fused epilogues (CSD_MODE_PROD).
//
// Replaces the cuBLAS calls of the block step:
//   * Q/K/V projections (model.cpp:63-70): ONE launch over the three weights, C = x W,
//     bf16 out in the token-major [B, N, H, E] layout the attention kernels read;
//   * output projection + residual (model.cpp:107-120, :200): x_mid = x + O Wo in the
//     epilogue (no x -> x_mid copy, no beta = 1 read-modify-write of a pre-copied C);
//   * dense MLP (mlp.cpp:49-81) as two TRANSPOSED GEMMs over the chunk-major activation
//     cache [B, C, F, chunk] the sparse-delta MLP keeps (north_star item 4/5):
//       up  : pre^T[f, r] = W1[f, :] . x[r, :]      (M = neurons, N = one chunk's rows)
//             epilogue: a = gelu(pre + b1[f]) -> cm[z, f, r] (one 2*chunk-byte run per
//             thread) — the bias/GELU pass and the [B*N, F] pre tensor disappear;
//       down: out^T[d, r] = W2[:, d]^T . cm[z, :, r] (A = W2 MN-major, B = the cache slab
//             MN-major)  epilogue: M_cache[r, d] = out + b2[d]; x_out = x_mid + M_cache.
//
// Tile 128 x BN (BN = 64..256, the chunk for the transposed GEMMs), K step 64 (one 128 B
// swizzle atom), a 4-6 stage TMA ring, fp32 accumulators double-buffered in TMEM so a
// tile's epilogue overlaps the next tile's main loop.  Roles: warp 0 lane 0 TMA producer,
// warp 1 MMA issuer (elected lane), warps 4-11 epilogue (two warps per TMEM lane quadrant,
// each owning half of the tile's columns).  Tiles are walked persistently with the index
// over the SMALLER operand varying fastest, so the larger operand's tiles are shared in L2
// by the CTAs running concurrently.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
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

enum : int { kEpiStore = 0, kEpiResid = 1, kEpiGeluCm = 2, kEpiMlpOut = 3, kEpiMlpRow = 4 };

constexpr uint32_t kGemmThreads = 384;
constexpr uint32_t kGemmMaxSmem = 227 * 1024;

struct GemmParams {
    int k;                   // contraction length (multiple of 64)
    int tiles_m, tiles_n;    // output tiles
    int n_fastest;           // tile order: n index varies fastest (A tiles reused in L2)
    int stages;
    uint32_t a_stage, b_stage;  // smem bytes per stage
    int b_batched;           // MN-major B from the chunk-major cache: rows nt * k + kk
    int n_split;             // kEpiStore over several weights: N tiles per weight (0: one)
    int n_total;             // kEpiStore / kEpiResid: output row pitch (elements)
    __nv_bfloat16* out0;
    __nv_bfloat16* out1;
    __nv_bfloat16* out2;
    const __nv_bfloat16* resid;  // kEpiResid
    const float* bias;           // kEpiGeluCm: b1[f]; kEpiMlpOut: b2[d]
    __nv_bfloat16* cm;           // kEpiGeluCm: [chunks][M][BN]
    float* mcache;               // kEpiMlpOut: [chunks * BN][M] fp32
    const __nv_bfloat16* xmid;   // kEpiMlpOut: residual in (nullable)
    __nv_bfloat16* xout;         // kEpiMlpOut: x_out = x_mid + M_cache (nullable)
    int m_total;                 // M (rows of A / leading dim of the MLP-out outputs)
    int chunk;                   // A from the chunk-major cache: rows per chunk
    int a_bk, a_brows;           // K-major A in column blocks of a_bk, stacked by rows (0: plain)
};

// Epilogue of one thread: 32-column chunks r[c * 32 ..] of tile row `m` (TMEM lane), tile
// column offset colbase within N tile nt.
template <int EPI, int kChunks, int BN>
__device__ __forceinline__ void gemm_epilogue(const GemmParams& p, int m, int nt, int colbase,
                                              const uint32_t* r) {
    if (EPI == kEpiStore || EPI == kEpiResid) {
        __nv_bfloat16* out = p.out0;
        int ncol0 = nt * BN;
        if (EPI == kEpiStore && p.n_split > 0) {
            const int which = nt / p.n_split;
            out = which == 0 ? p.out0 : which == 1 ? p.out1 : p.out2;
            ncol0 = (nt % p.n_split) * BN;
        }
        const int64_t o = (int64_t)m * p.n_total + ncol0 + colbase;
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
            uint4 rv[4];
            if (EPI == kEpiResid) {
                const uint4* rp = reinterpret_cast<const uint4*>(p.resid + o + c * 32);
#pragma unroll
                for (int u = 0; u < 4; ++u) rv[u] = rp[u];
            }
            uint4* dp = reinterpret_cast<uint4*>(out + o + c * 32);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                float f[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(r[c * 32 + u * 8 + e]);
                if (EPI == kEpiResid) {
                    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&rv[u]);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 x2 = __bfloat1622float2(h2[e]);
                        f[2 * e] += x2.x;
                        f[2 * e + 1] += x2.y;
                    }
                }
                dp[u] = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]),
                                   pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
            }
        }
    } else if (EPI == kEpiGeluCm) {
        // thread = neuron m of chunk nt: a = gelu(pre + b1) over the chunk's rows,
        // one contiguous run of the chunk-major cache
        const float b = p.bias[m];
        __nv_bfloat16* dst = p.cm + ((int64_t)nt * p.m_total + m) * BN + colbase;
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
            uint4* dp = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    w[e] = pack_bf16x2(gelu_tanh_approx(__uint_as_float(r[c * 32 + u * 8 + 2 * e]) + b),
                                       gelu_tanh_approx(__uint_as_float(r[c * 32 + u * 8 + 2 * e + 1]) + b));
                dp[u] = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
    } else if (EPI == kEpiMlpOut) {
        // kEpiMlpOut: thread = model dim m, columns = the chunk's rows; per row the
        // warp's 32 consecutive dims make 128 B (fp32) / 64 B (bf16) runs
        const float b = p.bias != nullptr ? p.bias[m] : 0.f;
        const int64_t row0 = (int64_t)nt * BN + colbase;
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
            __nv_bfloat16 xm[32];
            if (p.xout != nullptr) {
#pragma unroll
                for (int e = 0; e < 32; ++e)
                    xm[e] = p.xmid[(row0 + c * 32 + e) * p.m_total + m];
            }
#pragma unroll
            for (int e = 0; e < 32; ++e) {
                const float v = __uint_as_float(r[c * 32 + e]) + b;
                const int64_t o = (row0 + c * 32 + e) * p.m_total + m;
                p.mcache[o] = v;
                if (p.xout != nullptr) p.xout[o] = __float2bfloat16_rn(__bfloat162float(xm[e]) + v);
            }
        }
    }
    if (EPI == kEpiMlpRow) {
        // thread = token row m; columns = model dims (row-contiguous M_cache / x_out runs)
        const int64_t o = (int64_t)m * p.n_total + (int64_t)nt * BN + colbase;
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
            float4 bb[8];
            const float4* bp = reinterpret_cast<const float4*>(p.bias + (int64_t)nt * BN + colbase + c * 32);
#pragma unroll
            for (int u = 0; u < 8; ++u) bb[u] = p.bias != nullptr ? bp[u] : make_float4(0.f, 0.f, 0.f, 0.f);
            uint4 xv[4];
            if (p.xout != nullptr) {
                const uint4* xp = reinterpret_cast<const uint4*>(p.xmid + o + c * 32);
#pragma unroll
                for (int u = 0; u < 4; ++u) xv[u] = xp[u];
            }
            const float* bf = reinterpret_cast<const float*>(bb);
            float v[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[c * 32 + e]) + bf[e];
            float4* mp = reinterpret_cast<float4*>(p.mcache + o + c * 32);
#pragma unroll
            for (int u = 0; u < 8; ++u) mp[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
            if (p.xout != nullptr) {
                uint4* xo = reinterpret_cast<uint4*>(p.xout + o + c * 32);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&xv[u]);
                    uint32_t w[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 x2 = __bfloat1622float2(h2[e]);
                        w[e] = pack_bf16x2(x2.x + v[8 * u + 2 * e], x2.y + v[8 * u + 2 * e + 1]);
                    }
                    xo[u] = make_uint4(w[0], w[1], w[2], w[3]);
                }
            }
        }
    }
}

template <int BN, bool AMN, bool BMN, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
k_gemm_tc(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b0,
          const __grid_constant__ CUtensorMap tm_b1, const __grid_constant__ CUtensorMap tm_b2,
          const GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_u32 = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = p.stages;
    uint8_t* sa = smem;
    uint8_t* sb = smem + S * p.a_stage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * (p.a_stage + p.b_stage));
    uint64_t* full = bars;             // [S]
    uint64_t* empty = bars + S;        // [S]
    uint64_t* acc_full = bars + 2 * S;   // [2]
    uint64_t* acc_empty = bars + 2 * S + 2;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(acc_full + b, 1);
            mbar_init(acc_empty + b, 256);
        }
        fence_barrier_init();
    }
    constexpr uint32_t kTmemCols = 2 * BN <= 256 ? 256 : 512;
    if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    if (threadIdx.x == 0) pdl_trigger();
    const int ntiles = p.tiles_m * p.tiles_n;
    const int kblocks = p.k / 64;
    auto tile_mn = [&](int t, int& mt, int& nt) {
        if (p.n_fastest) {
            nt = t % p.tiles_n;
            mt = t / p.tiles_n;
        } else {
            mt = t % p.tiles_m;
            nt = t / p.tiles_m;
        }
    };

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------------------ TMA producer
            tma_prefetch_desc(&tm_a);
            tma_prefetch_desc(&tm_b0);
            uint32_t it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int mt, nt;
                tile_mn(t, mt, nt);
                const CUtensorMap* tb = &tm_b0;
                int nt_local = nt;
                if (p.n_split > 0) {
                    const int which = nt / p.n_split;
                    tb = which == 0 ? &tm_b0 : which == 1 ? &tm_b1 : &tm_b2;
                    nt_local = nt % p.n_split;
                }
                for (int kb = 0; kb < kblocks; ++kb, ++it) {
                    const uint32_t s = it % S, ph = (it / S) & 1;
                    if (it >= (uint32_t)S) mbar_wait(empty + s, ph ^ 1);
                    mbar_arrive_expect_tx(full + s, p.a_stage + p.b_stage);
                    uint8_t* a_dst = sa + s * p.a_stage;
                    uint8_t* b_dst = sb + s * p.b_stage;
                    if (!AMN) {
                        if (p.a_bk > 0)  // block (kb * 64) / a_bk of the row-stacked A
                            tma_load_2d(&tm_a, full + s, a_dst, (kb * 64) % p.a_bk,
                                        ((kb * 64) / p.a_bk) * p.a_brows + mt * 128);
                        else
                            tma_load_2d(&tm_a, full + s, a_dst, kb * 64, mt * 128);
                    } else {
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            tma_load_2d(&tm_a, full + s, a_dst + h * 8192, mt * 128 + 64 * h, kb * 64);
                    }
                    if (!BMN) {
                        tma_load_2d(tb, full + s, b_dst, kb * 64, nt_local * BN);
                    } else {
                        const int col0 = p.b_batched ? 0 : nt_local * BN;
                        const int row0 = (p.b_batched ? nt * p.k : 0) + kb * 64;
#pragma unroll
                        for (int h = 0; h < BN / 64; ++h)
                            tma_load_2d(tb, full + s, b_dst + h * 8192, col0 + 64 * h, row0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA issuer
        constexpr uint32_t idesc = idesc_bf16(128, BN, AMN, BMN);
        const uint32_t sA = smem_u32(sa), sB = smem_u32(sb);
        uint32_t it = 0, i = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const uint32_t buf = i & 1;
            if (i >= 2) mbar_wait(acc_empty + buf, ((i >> 1) - 1) & 1);
            tc_fence_after();
            const uint32_t dt = tmem + buf * BN;
            for (int kb = 0; kb < kblocks; ++kb, ++it) {
                const uint32_t s = it % S, ph = (it / S) & 1;
                mbar_wait(full + s, ph);
                tc_fence_after();
                const uint32_t a0 = sA + s * p.a_stage, b0 = sB + s * p.b_stage;
                uint64_t da[4], db[4];
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    da[kk] = AMN ? desc_mnmajor_sw128(a0 + kk * 2048, 8192) : desc_kmajor_sw128(a0 + kk * 32);
                    db[kk] = BMN ? desc_mnmajor_sw128(b0 + kk * 2048, 8192) : desc_kmajor_sw128(b0 + kk * 32);
                }
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_bf16(dt, da[kk], db[kk], idesc, (kb | kk) ? 1u : 0u);
                    mma_commit(empty + s);
                }
                __syncwarp();
            }
            if (elect_one()) mma_commit(acc_full + buf);
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ---------------------------------------------------------------- epilogue
        const int q = warp & 3, half = (warp - 4) >> 2;
        constexpr int kChunks = BN / 64;  // 32-column chunks per half
        const int row = q * 32 + lane;     // TMEM lane = tile row
        uint32_t i = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            int mt, nt;
            tile_mn(t, mt, nt);
            const uint32_t buf = i & 1;
            mbar_wait(acc_full + buf, (i >> 1) & 1);
            tc_fence_after();
            uint32_t r[kChunks * 32];
#pragma unroll
            for (int c = 0; c < kChunks; ++c)
                tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + buf * BN + half * (BN / 2) + c * 32,
                          *reinterpret_cast<uint32_t(*)[32]>(&r[c * 32]));
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(acc_empty + buf);  // TMEM buffer free: the next tile's MMAs may start
            gemm_epilogue<EPI, kChunks, BN>(p, mt * 128 + row, nt, half * (BN / 2), r);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
}

// CTA-pair variant (cta_group::2): the pair computes a 256 x BN tile, CTA `rank` holding A
// rows [128 rank, +128) and B's N-half [BN/2 rank, +BN/2) -- 32 KB of operands per k step
// per SM instead of 48 KB (the single-CTA kernel is bound by the SM's L2 -> smem port).  The
// leader (rank 0) issues the MMAs (M = 256) and commits to both CTAs' barriers; both CTAs'
// TMA bytes land on the leader's full barrier; both epilogues release the accumulator on
// the leader's empty barrier.  ACM: A is MN-major from the chunk-major activation cache
// (cm[z][k][r], 64-row atoms never straddle a chunk).
template <int BN, bool BMN, int EPI, bool ACM>
__global__ void __launch_bounds__(kGemmThreads, 1)
k_gemm2_tc(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b0,
           const __grid_constant__ CUtensorMap tm_b1, const __grid_constant__ CUtensorMap tm_b2,
           const GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_u32 = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int S = p.stages;
    uint8_t* sa = smem;
    uint8_t* sb = smem + S * p.a_stage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * (p.a_stage + p.b_stage));
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* acc_full = bars + 2 * S;
    uint64_t* acc_empty = bars + 2 * S + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(acc_full + b, 1);
            mbar_init(acc_empty + b, 16);  // 8 epilogue warps x 2 CTAs (leader's copy counts)
        }
        fence_barrier_init();
    }
    constexpr uint32_t kTmemCols = 2 * BN <= 256 ? 256 : 512;
    if (warp == 1) tmem_alloc_pair<kTmemCols>(tmem_slot);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    if (threadIdx.x == 0) pdl_trigger();
    const int ntiles = p.tiles_m * p.tiles_n;  // tiles_m counts 256-row pair tiles
    const int kblocks = p.k / 64;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    auto tile_mn = [&](int t, int& mt, int& nt) {
        if (p.n_fastest) {
            nt = t % p.tiles_n;
            mt = t / p.tiles_n;
        } else {
            mt = t % p.tiles_m;
            nt = t / p.tiles_m;
        }
    };
    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------------------ TMA producer
            tma_prefetch_desc(&tm_a);
            tma_prefetch_desc(&tm_b0);
            uint32_t it = 0;
            for (int t = pair; t < ntiles; t += npairs) {
                int mt, nt;
                tile_mn(t, mt, nt);
                const CUtensorMap* tb = &tm_b0;
                int nt_local = nt;
                if (p.n_split > 0) {
                    const int which = nt / p.n_split;
                    tb = which == 0 ? &tm_b0 : which == 1 ? &tm_b1 : &tm_b2;
                    nt_local = nt % p.n_split;
                }
                const int m_cta = mt * 256 + (int)rank * 128;
                const int n_cta = nt_local * BN + (int)rank * (BN / 2);
                for (int kb = 0; kb < kblocks; ++kb, ++it) {
                    const uint32_t s = it % S, ph = (it / S) & 1;
                    if (it >= (uint32_t)S) mbar_wait(empty + s, ph ^ 1);
                    if (rank == 0) mbar_arrive_expect_tx(full + s, 2 * (p.a_stage + p.b_stage));
                    uint8_t* a_dst = sa + s * p.a_stage;
                    uint8_t* b_dst = sb + s * p.b_stage;
                    if (!ACM) {
                        if (p.a_bk > 0)
                            tma_load_2d_pair(&tm_a, full + s, a_dst, (kb * 64) % p.a_bk,
                                             ((kb * 64) / p.a_bk) * p.a_brows + m_cta);
                        else
                            tma_load_2d_pair(&tm_a, full + s, a_dst, kb * 64, m_cta);
                    } else {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int m = m_cta + 64 * h;
                            tma_load_2d_pair(&tm_a, full + s, a_dst + h * 8192, m % p.chunk,
                                             (m / p.chunk) * p.k + kb * 64);
                        }
                    }
                    if (!BMN) {
                        tma_load_2d_pair(tb, full + s, b_dst, kb * 64, n_cta);
                    } else {
#pragma unroll
                        for (int h = 0; h < BN / 128; ++h)
                            tma_load_2d_pair(tb, full + s, b_dst + h * 8192, n_cta + 64 * h, kb * 64);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            // ------------------------------------------------------------ MMA issuer (leader)
            constexpr uint32_t idesc = idesc_bf16(256, BN, ACM, BMN);
            const uint32_t sA = smem_u32(sa), sB = smem_u32(sb);
            uint32_t it = 0, i = 0;
            for (int t = pair; t < ntiles; t += npairs, ++i) {
                const uint32_t buf = i & 1;
                if (i >= 2) mbar_wait(acc_empty + buf, ((i >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t dt = tmem + buf * BN;
                for (int kb = 0; kb < kblocks; ++kb, ++it) {
                    const uint32_t s = it % S, ph = (it / S) & 1;
                    mbar_wait(full + s, ph);
                    tc_fence_after();
                    const uint32_t a0 = sA + s * p.a_stage, b0 = sB + s * p.b_stage;
                    uint64_t da[4], db[4];
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        da[kk] = ACM ? desc_mnmajor_sw128(a0 + kk * 2048, 8192) : desc_kmajor_sw128(a0 + kk * 32);
                        db[kk] = BMN ? desc_mnmajor_sw128(b0 + kk * 2048, 8192) : desc_kmajor_sw128(b0 + kk * 32);
                    }
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_bf16_pair(dt, da[kk], db[kk], idesc, (kb | kk) ? 1u : 0u);
                        mma_commit_pair(empty + s);
                    }
                    __syncwarp();
                }
                if (elect_one()) mma_commit_pair(acc_full + buf);
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        // ---------------------------------------------------------------- epilogue
        const int q = warp & 3, half = (warp - 4) >> 2;
        constexpr int kChunks = BN / 64;
        const int row = q * 32 + lane;
        uint32_t i = 0;
        for (int t = pair; t < ntiles; t += npairs, ++i) {
            int mt, nt;
            tile_mn(t, mt, nt);
            const uint32_t buf = i & 1;
            mbar_wait(acc_full + buf, (i >> 1) & 1);
            tc_fence_after();
            uint32_t r[kChunks * 32];
#pragma unroll
            for (int c = 0; c < kChunks; ++c)
                tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + buf * BN + half * (BN / 2) + c * 32,
                          *reinterpret_cast<uint32_t(*)[32]>(&r[c * 32]));
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            // the leader's barrier; release.cta is enough (the TMEM reads are waited and fenced),
            // release.cluster would cost a MEMBAR.ALL.GPU behind the previous tile's stores
            if (lane == 0) mbar_arrive_remote(acc_empty + buf, 0);
            gemm_epilogue<EPI, kChunks, BN>(p, mt * 256 + (int)rank * 128 + row, nt, half * (BN / 2), r);
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair<kTmemCols>(tmem);
    }
}

template <int BN, bool BMN, int EPI, bool ACM>
cudaError_t launch_gemm2(const CUtensorMap& ta, const CUtensorMap& tb0, const CUtensorMap& tb1,
                         const CUtensorMap& tb2, GemmParams p, cudaStream_t s) {
    p.a_stage = 128 * 128;
    p.b_stage = (BN / 2) * 128;
    const uint32_t stage = p.a_stage + p.b_stage;
    p.stages = (int)std::min<uint32_t>(8, (kGemmMaxSmem - 1024) / stage);
    const uint32_t smem = p.stages * stage + 256;
    auto kern = k_gemm2_tc<BN, BMN, EPI, ACM>;
    cudaError_t err = ensure_smem_attr(kern, (int)kGemmMaxSmem);
    if (err != cudaSuccess) return err;
    const int tiles = p.tiles_m * p.tiles_n;
    const int grid = std::min(2 * tiles, sm_count() & ~1);
    return launch_ex(kern, dim3((unsigned)grid), dim3(kGemmThreads), smem, s, 2, ta, tb0, tb1, tb2, p);
}

struct GemmShape {
    int bn;
    bool amn, bmn;
    int epi;
};

template <int BN, bool AMN, bool BMN, int EPI>
cudaError_t launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb0, const CUtensorMap& tb1,
                        const CUtensorMap& tb2, GemmParams p, cudaStream_t s) {
    p.a_stage = 128 * 128;
    p.b_stage = BN * 128;
    const uint32_t stage = p.a_stage + p.b_stage;
    p.stages = (int)std::min<uint32_t>(6, (kGemmMaxSmem - 1024) / stage);
    const uint32_t smem = p.stages * stage + 256;
    auto kern = k_gemm_tc<BN, AMN, BMN, EPI>;
    cudaError_t err = ensure_smem_attr(kern, (int)kGemmMaxSmem);
    if (err != cudaSuccess) return err;
    const int tiles = p.tiles_m * p.tiles_n;
    const unsigned grid = (unsigned)std::min(tiles, sm_count());
    return launch_ex(kern, dim3(grid), dim3(kGemmThreads), smem, s, 1, ta, tb0, tb1, tb2, p);
}

// 2-D bf16 map with an explicit box (columns x rows), 128 B swizzle.
bool map_box(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch,
             uint32_t box_cols, uint32_t box_rows);

}  // namespace

}  // namespace dev
}  // namespace csd

// --------------------------------------------------------------------------- host API
namespace csd {
namespace dev {

namespace {
bool map_box(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch,
             uint32_t box_cols, uint32_t box_rows) {
    (void)box_cols;  // always 64 (one 128 B swizzle row)
    return make_map_bf16(m, base, cols, rows, pitch, box_rows);
}
}  // namespace

bool gemm_tc_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("CSD_GEMM");
        return !(e != nullptr && std::string(e) == "cublas");
    }();
    return on;
}

// CTA-pair kernels (cta_group::2) where the shape allows; CSD_GEMM_PAIR=0 forces the
// single-CTA kernels.
static bool use_pair() {
    static const bool on = [] {
        const char* e = std::getenv("CSD_GEMM_PAIR");
        return !(e != nullptr && std::string(e) == "0");
    }();
    return on;
}

bool gemm_tc_proj_supported(int64_t rows, int64_t k, int64_t n) {
    return rows % 128 == 0 && k % 64 == 0 && n % 64 == 0 && rows >= 128;
}

static int proj_bn(int64_t n) {
    for (int bn : {256, 192, 128, 64})
        if (n % bn == 0) return bn;
    return 0;
}

// q|k|v[rows, n] = x[rows, k] @ {wq, wk, wv}[k, n]  (any of the outputs may be null: fewer
// weights); one launch.
static cudaError_t gemm_tc_proj_impl(const void* x, const void* const w[3], void* const out[3],
                                     int nw, int64_t rows, int64_t k, int64_t n, const void* resid,
                                     int64_t a_bk, cudaStream_t s) {
    if (!gemm_tc_proj_supported(rows, k, n) || nw < 1 || nw > 3) return cudaErrorNotSupported;
    if (a_bk > 0 && (a_bk % 64 || k % a_bk)) return cudaErrorNotSupported;
    const int bn = proj_bn(n);
    CUtensorMap ta, tb[3];
    // plain A [rows][k], or k / a_bk column blocks of width a_bk stacked by rows
    if (a_bk > 0 ? !map_box(&ta, x, a_bk, (k / a_bk) * rows, a_bk, 64, 128)
                 : !map_box(&ta, x, k, rows, k, 64, 128))
        return cudaErrorInvalidValue;
    for (int i = 0; i < 3; ++i)
        if (!map_box(&tb[i], w[i < nw ? i : 0], n, k, n, 64, 64)) return cudaErrorInvalidValue;
    GemmParams p{};
    p.k = (int)k;
    p.tiles_m = (int)(rows / 128);
    p.tiles_n = (int)(n / bn) * nw;
    // A = activations, B = weights: reuse the larger operand's tiles across the fast index
    p.n_fastest = (rows * k > k * n * nw) ? 1 : 0;
    p.n_split = nw > 1 ? (int)(n / bn) : 0;
    p.n_total = (int)n;
    p.out0 = static_cast<__nv_bfloat16*>(out[0]);
    p.out1 = static_cast<__nv_bfloat16*>(out[nw > 1 ? 1 : 0]);
    p.out2 = static_cast<__nv_bfloat16*>(out[nw > 2 ? 2 : 0]);
    p.resid = static_cast<const __nv_bfloat16*>(resid);
    p.m_total = (int)rows;
    p.a_bk = (int)a_bk;
    p.a_brows = (int)rows;
    if (use_pair() && rows % 256 == 0 && bn % 128 == 0) {
        p.tiles_m = (int)(rows / 256);
        if (resid != nullptr) {
            if (nw != 1) return cudaErrorInvalidValue;
            return bn == 256 ? launch_gemm2<256, true, kEpiResid, false>(ta, tb[0], tb[1], tb[2], p, s)
                             : launch_gemm2<128, true, kEpiResid, false>(ta, tb[0], tb[1], tb[2], p, s);
        }
        return bn == 256 ? launch_gemm2<256, true, kEpiStore, false>(ta, tb[0], tb[1], tb[2], p, s)
                         : launch_gemm2<128, true, kEpiStore, false>(ta, tb[0], tb[1], tb[2], p, s);
    }
    if (resid != nullptr) {
        if (nw != 1) return cudaErrorInvalidValue;
        switch (bn) {
            case 256: return launch_gemm<256, false, true, kEpiResid>(ta, tb[0], tb[1], tb[2], p, s);
            case 192: return launch_gemm<192, false, true, kEpiResid>(ta, tb[0], tb[1], tb[2], p, s);
            case 128: return launch_gemm<128, false, true, kEpiResid>(ta, tb[0], tb[1], tb[2], p, s);
            default: return launch_gemm<64, false, true, kEpiResid>(ta, tb[0], tb[1], tb[2], p, s);
        }
    }
    switch (bn) {
        case 256: return launch_gemm<256, false, true, kEpiStore>(ta, tb[0], tb[1], tb[2], p, s);
        case 192: return launch_gemm<192, false, true, kEpiStore>(ta, tb[0], tb[1], tb[2], p, s);
        case 128: return launch_gemm<128, false, true, kEpiStore>(ta, tb[0], tb[1], tb[2], p, s);
        default: return launch_gemm<64, false, true, kEpiStore>(ta, tb[0], tb[1], tb[2], p, s);
    }
}

cudaError_t gemm_tc_proj(const void* x, const void* const w[3], void* const out[3], int nw,
                         int64_t rows, int64_t k, int64_t n, const void* resid, cudaStream_t s) {
    return gemm_tc_proj_impl(x, w, out, nw, rows, k, n, resid, 0, s);
}

// out[rows, n] = resid + A @ w with A given as k / a_bk column blocks [k / a_bk][rows][a_bk]
// (the head-sharded attention outputs after the token all-to-all)
cudaError_t gemm_tc_proj_blocked(const void* a_blocks, const void* w, void* out, int64_t rows,
                                 int64_t k, int64_t n, const void* resid, int64_t a_bk,
                                 int64_t a_brows, cudaStream_t s) {
    if (a_brows != rows) return cudaErrorInvalidValue;
    const void* ws[3] = {w, w, w};
    void* os[3] = {out, out, out};
    return gemm_tc_proj_impl(a_blocks, ws, os, 1, rows, k, n, resid, a_bk, s);
}

bool gemm_tc_mlp_supported(int64_t d, int64_t f, int64_t chunk) {
    return d % 128 == 0 && f % 128 == 0 && (chunk == 64 || chunk == 128 || chunk == 192 || chunk == 256);
}

// cm[z, f, r] = gelu(sum_d x[z*chunk + r, d] W1[f, d] + b1[f])  for every chunk z
cudaError_t gemm_tc_mlp_up(const void* x, const void* w1, const float* b1, int64_t chunks,
                           int64_t chunk, int64_t d, int64_t f, void* cm, cudaStream_t s) {
    if (!gemm_tc_mlp_supported(d, f, chunk)) return cudaErrorNotSupported;
    CUtensorMap ta, tb;
    if (!map_box(&ta, w1, d, f, d, 64, 128) ||
        !map_box(&tb, x, d, chunks * chunk, d, 64, (uint32_t)chunk))
        return cudaErrorInvalidValue;
    GemmParams p{};
    p.k = (int)d;
    p.tiles_m = (int)(f / 128);
    p.tiles_n = (int)chunks;
    p.n_fastest = (f * d > chunks * chunk * d) ? 1 : 0;
    p.bias = b1;
    p.cm = static_cast<__nv_bfloat16*>(cm);
    p.m_total = (int)f;
    if (use_pair() && f % 256 == 0) {
        // CTA pairs: 256 neurons x one chunk per pair, each CTA stages half the chunk's rows
        CUtensorMap tb2;
        if (!map_box(&tb2, x, d, chunks * chunk, d, 64, (uint32_t)(chunk / 2))) return cudaErrorInvalidValue;
        p.tiles_m = (int)(f / 256);
        switch (chunk) {
            case 256: return launch_gemm2<256, false, kEpiGeluCm, false>(ta, tb2, tb2, tb2, p, s);
            case 192: return launch_gemm2<192, false, kEpiGeluCm, false>(ta, tb2, tb2, tb2, p, s);
            case 128: return launch_gemm2<128, false, kEpiGeluCm, false>(ta, tb2, tb2, tb2, p, s);
            default: return launch_gemm2<64, false, kEpiGeluCm, false>(ta, tb2, tb2, tb2, p, s);
        }
    }
    switch (chunk) {
        case 256: return launch_gemm<256, false, false, kEpiGeluCm>(ta, tb, tb, tb, p, s);
        case 192: return launch_gemm<192, false, false, kEpiGeluCm>(ta, tb, tb, tb, p, s);
        case 128: return launch_gemm<128, false, false, kEpiGeluCm>(ta, tb, tb, tb, p, s);
        default: return launch_gemm<64, false, false, kEpiGeluCm>(ta, tb, tb, tb, p, s);
    }
}

// M_cache[z*chunk + r, dd] = sum_f cm[z, f, r] W2[f, dd] + b2[dd];  x_out = x_mid + M_cache
cudaError_t gemm_tc_mlp_down(const void* cm, const void* w2, const float* b2, int64_t chunks,
                             int64_t chunk, int64_t d, int64_t f, float* mcache,
                             const void* x_mid, void* x_out, cudaStream_t s) {
    if (!gemm_tc_mlp_supported(d, f, chunk)) return cudaErrorNotSupported;
    if (use_pair() && (chunks * chunk) % 256 == 0 && d % 256 == 0 && chunk % 64 == 0) {
        // CTA pairs, token-major: out[r, dd] over 256 rows x 256 dims per pair; A = the
        // chunk-major cache read MN-major (64-row atoms of one chunk), B = W2 [F, D] MN-major
        CUtensorMap ta, tb;
        if (!map_box(&ta, cm, chunk, chunks * f, chunk, 64, 64) || !map_box(&tb, w2, d, f, d, 64, 64))
            return cudaErrorInvalidValue;
        GemmParams p{};
        p.k = (int)f;
        p.chunk = (int)chunk;
        p.tiles_m = (int)(chunks * chunk / 256);
        p.tiles_n = (int)(d / 256);
        p.n_fastest = 0;  // the cache (A) is the larger operand... both are read per tile row
        p.n_total = (int)d;
        p.bias = b2;
        p.mcache = mcache;
        p.xmid = static_cast<const __nv_bfloat16*>(x_mid);
        p.xout = static_cast<__nv_bfloat16*>(x_out);
        p.m_total = (int)(chunks * chunk);
        return launch_gemm2<256, true, kEpiMlpRow, true>(ta, tb, tb, tb, p, s);
    }
    CUtensorMap ta, tb;
    if (!map_box(&ta, w2, d, f, d, 64, 64) ||
        !map_box(&tb, cm, chunk, chunks * f, chunk, 64, 64))
        return cudaErrorInvalidValue;
    GemmParams p{};
    p.k = (int)f;
    p.tiles_m = (int)(d / 128);
    p.tiles_n = (int)chunks;
    p.n_fastest = (d * f > chunks * chunk * f) ? 1 : 0;
    p.b_batched = 1;
    p.bias = b2;
    p.mcache = mcache;
    p.xmid = static_cast<const __nv_bfloat16*>(x_mid);
    p.xout = static_cast<__nv_bfloat16*>(x_out);
    p.m_total = (int)d;
    switch (chunk) {
        case 256: return launch_gemm<256, true, true, kEpiMlpOut>(ta, tb, tb, tb, p, s);
        case 192: return launch_gemm<192, true, true, kEpiMlpOut>(ta, tb, tb, tb, p, s);
        case 128: return launch_gemm<128, true, true, kEpiMlpOut>(ta, tb, tb, tb, p, s);
        default: return launch_gemm<64, true, true, kEpiMlpOut>(ta, tb, tb, tb, p, s);
    }
}

}  // namespace dev
}  // namespace csd
