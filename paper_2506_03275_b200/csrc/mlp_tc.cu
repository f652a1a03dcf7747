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
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace csd {
namespace dev {

using namespace csd::tc;

bool make_map_bf16(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows,
                   uint64_t pitch_elems, uint32_t box_rows);

constexpr int kMlpStages = 2;  // 2 x 48 KB: two CTAs per SM (grid tails, TMA overlap)
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
    const int32_t* idx;
    const int32_t* counts;
    int k_max, k_pad;
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
                                          uint64_t*& done, uint32_t& tmem) {
    using L = MlpLayout<NT>;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
    full = bars;
    empty = bars + kMlpStages;
    done = bars + 2 * kMlpStages;
    uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 2 * kMlpStages + 1);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kMlpStages; ++s) {
            mbar_init(full + s, 1);
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
template <int NT>
__global__ void __launch_bounds__(MlpLayout<NT>::kThreads, 2)
k_smlp_up(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w1g,
          const MlpParams p) {
    using L = MlpLayout<NT>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int z = blockIdx.y, tn = blockIdx.x;
    const int cnt = p.counts[z];
    if (tn * 128 >= cnt) return;
    const int b = z / p.chunks, c = z % p.chunks;
    const int x_row0 = b * p.n + c * p.chunk;
    const int kblocks = p.d / 64;
    const int32_t* ids = p.idx + (int64_t)z * p.k_max;

    uint64_t *full, *empty, *done;
    uint32_t tmem;
    mlp_setup<NT>(smem, full, empty, done, tmem);

    if (warp == 0 || warp == 2 || warp == 3) {
        // producers: warp 0 issues the x tiles; the 32 W1-row gather4s per stage are spread
        // over warps 0/2/3 (one warp's TMA issue is serialised, scripts/gather_bench.cu)
        const int pw = warp == 0 ? 0 : warp - 1;
        const bool mine = (lane % 3) == pw;
        int32_t rows[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int nn = tn * 128 + lane * 4 + i;
            rows[i] = ids[nn < cnt ? nn : cnt - 1];
        }
        if (warp == 0 && lane == 0) {
            tma_prefetch_desc(&tm_x);
            tma_prefetch_desc(&tm_w1g);
        }
        for (int kb = 0; kb < kblocks; ++kb) {
            const int s = kb % kMlpStages;
            if (kb >= kMlpStages) mbar_wait(empty + s, ((kb / kMlpStages) - 1) & 1);
            if (warp == 0 && lane == 0) {
                mbar_arrive_expect_tx(full + s, (NT + 1) * kTile);
                for (int t = 0; t < NT; ++t)
                    tma_load_2d(&tm_x, full + s, smem + L::kA + (s * NT + t) * kTile, kb * 64,
                                x_row0 + t * 128);
            }
            if (mine)
                tma_gather4(&tm_w1g, full + s, smem + L::kB + s * kTile + lane * 512, kb * 64,
                            rows[0], rows[1], rows[2], rows[3]);
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t id = idesc_bf16(128, 128, false, false);
            const uint32_t sA = smem_u32(smem + L::kA), sB = smem_u32(smem + L::kB);
            for (int kb = 0; kb < kblocks; ++kb) {
                const int s = kb % kMlpStages;
                mbar_wait(full + s, (kb / kMlpStages) & 1);
                tc_fence_after();
                for (int t = 0; t < NT; ++t) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_bf16(tmem + t * 128, desc_kmajor_sw128(sA + (s * NT + t) * kTile + kk * 32),
                                 desc_kmajor_sw128(sB + s * kTile + kk * 32), id,
                                 (kb > 0 || kk > 0) ? 1u : 0u);
                }
                mma_commit(empty + s);
            }
            mma_commit(done);
        }
    } else if (warp >= 4) {
        const int sw = warp - 4, t = sw >> 2, quad = warp & 3;
        const int r = t * 128 + quad * 32 + lane;  // row within the chunk
        const bool row_ok = r < p.chunk;
        // stage this tile's neuron ids and biases in smem while the MMAs run, so the
        // epilogue's cache read-modify-write has no dependent global loads
        int32_t* s_ids = reinterpret_cast<int32_t*>(smem + L::kBar + 128);
        float* s_b1 = reinterpret_cast<float*>(smem + L::kBar + 128 + 512);
        const int et = sw * 32 + lane;
        if (et < 128) {
            const int nn = tn * 128 + et;
            const int neuron = ids[nn < cnt ? nn : cnt - 1];
            s_ids[et] = neuron;
            s_b1[et] = p.b1[neuron];
        }
        named_bar_sync(1, 128 * NT);
        mbar_wait(done, 0);
        tc_fence_after();
        const uint32_t tacc = tmem + ((uint32_t)(quad * 32) << 16) + t * 128;
        __nv_bfloat16* drow = p.delta + ((int64_t)z * p.chunk + r) * p.k_pad + tn * 128;
        __nv_bfloat16* __restrict__ cache_base = p.act_cm + (int64_t)z * p.f * p.chunk + r;
#pragma unroll 1
        for (int cc = 0; cc < 4; ++cc) {
            uint32_t acc[32];
            tmem_ld32(tacc + cc * 32, acc);
            tmem_ld_wait();
            if (!row_ok) continue;
            const int nvalid = min(32, cnt - (tn * 128 + cc * 32));
            float old[32], dl[32];
#pragma unroll
            for (int i = 0; i < 32; ++i)  // all loads first (independent)
                old[i] = i < nvalid ? __bfloat162float(cache_base[(int64_t)s_ids[cc * 32 + i] * p.chunk])
                                    : 0.f;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                dl[i] = 0.f;
                if (i < nvalid) {
                    const float a = fast_gelu(__uint_as_float(acc[i]) + s_b1[cc * 32 + i]);
                    const __nv_bfloat16 a16 = __float2bfloat16_rn(a);
                    cache_base[(int64_t)s_ids[cc * 32 + i] * p.chunk] = a16;
                    dl[i] = __bfloat162float(a16) - old[i];
                }
            }
            uint4* dst = reinterpret_cast<uint4*>(drow + cc * 32);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint4 v;
                v.x = pack_bf16x2(dl[q * 8 + 0], dl[q * 8 + 1]);
                v.y = pack_bf16x2(dl[q * 8 + 2], dl[q * 8 + 3]);
                v.z = pack_bf16x2(dl[q * 8 + 4], dl[q * 8 + 5]);
                v.w = pack_bf16x2(dl[q * 8 + 6], dl[q * 8 + 7]);
                dst[q] = v;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<L::kTmemCols>(tmem);
    }
}

// ------------------------------------------------------------------ down projection
template <int NT>
__global__ void __launch_bounds__(MlpLayout<NT>::kThreads, 2)
k_smlp_down(const __grid_constant__ CUtensorMap tm_delta,
            const __grid_constant__ CUtensorMap tm_w2g, const MlpParams p) {
    using L = MlpLayout<NT>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int z = blockIdx.y, td = blockIdx.x;
    const int cnt = p.counts[z];
    const int b = z / p.chunks, c = z % p.chunks;
    if (cnt == 0) {  // no recomputed neurons: M_cache unchanged, only the residual
        if (p.x_out != nullptr) {
            for (int r = threadIdx.x; r < p.chunk; r += blockDim.x) {
                const int64_t row = (int64_t)b * p.n + (int64_t)c * p.chunk + r;
                for (int cc = 0; cc < 4; ++cc) {
                    float m[32];
                    const float* src = p.out_cache + row * p.d + td * 128 + cc * 32;
#pragma unroll
                    for (int i = 0; i < 32; ++i) m[i] = src[i];
                    residual32(p, row, td * 128 + cc * 32, m);
                }
            }
        }
        return;
    }
    const int kblocks = (cnt + 63) / 64;
    const int32_t* ids = p.idx + (int64_t)z * p.k_max;

    uint64_t *full, *empty, *done;
    uint32_t tmem;
    mlp_setup<NT>(smem, full, empty, done, tmem);

    if (warp == 0 || warp == 2 || warp == 3) {
        const int pw = warp == 0 ? 0 : warp - 1;
        const bool mine = (lane % 3) == pw;
        if (warp == 0 && lane == 0) {
            tma_prefetch_desc(&tm_delta);
            tma_prefetch_desc(&tm_w2g);
        }
        const int strip = lane >> 4, g4 = lane & 15;  // 16 lanes x 4 rows per 64-column strip
        for (int kb = 0; kb < kblocks; ++kb) {
            const int s = kb % kMlpStages;
            int32_t rows[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                int nn = kb * 64 + g4 * 4 + i;
                rows[i] = ids[nn < cnt ? nn : cnt - 1];
            }
            if (kb >= kMlpStages) mbar_wait(empty + s, ((kb / kMlpStages) - 1) & 1);
            if (warp == 0 && lane == 0) {
                mbar_arrive_expect_tx(full + s, (NT + 1) * kTile);
                for (int t = 0; t < NT; ++t)
                    tma_load_2d(&tm_delta, full + s, smem + L::kA + (s * NT + t) * kTile, kb * 64,
                                z * p.chunk + t * 128);
            }
            // B tile: 64 neuron rows x 128 D columns as two 64-column (128 B) strips of 8 KB
            if (mine)
                tma_gather4(&tm_w2g, full + s, smem + L::kB + s * kTile + strip * 8192 + g4 * 512,
                            td * 128 + strip * 64, rows[0], rows[1], rows[2], rows[3]);
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t id = idesc_bf16(128, 128, false, true);
            const uint32_t sA = smem_u32(smem + L::kA), sB = smem_u32(smem + L::kB);
            for (int kb = 0; kb < kblocks; ++kb) {
                const int s = kb % kMlpStages;
                mbar_wait(full + s, (kb / kMlpStages) & 1);
                tc_fence_after();
                for (int t = 0; t < NT; ++t) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_bf16(tmem + t * 128, desc_kmajor_sw128(sA + (s * NT + t) * kTile + kk * 32),
                                 desc_mnmajor_sw128(sB + s * kTile + kk * 2048, 8192), id,
                                 (kb > 0 || kk > 0) ? 1u : 0u);
                }
                mma_commit(empty + s);
            }
            mma_commit(done);
        }
    } else if (warp >= 4) {
        const int sw = warp - 4, t = sw >> 2, quad = warp & 3;
        const int r = t * 128 + quad * 32 + lane;
        const bool row_ok = r < p.chunk;
        mbar_wait(done, 0);
        tc_fence_after();
        const uint32_t tacc = tmem + ((uint32_t)(quad * 32) << 16) + t * 128;
        float* orow = p.out_cache + ((int64_t)b * p.n + (int64_t)c * p.chunk + r) * p.d + td * 128;
#pragma unroll 1
        for (int cc = 0; cc < 4; ++cc) {
            uint32_t acc[32];
            tmem_ld32(tacc + cc * 32, acc);
            tmem_ld_wait();
            if (!row_ok) continue;
            float4* o4 = reinterpret_cast<float4*>(orow + cc * 32);
            float m[32];
            float4 v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = o4[q];  // batch the loads
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                v[q].x += __uint_as_float(acc[q * 4 + 0]);
                v[q].y += __uint_as_float(acc[q * 4 + 1]);
                v[q].z += __uint_as_float(acc[q * 4 + 2]);
                v[q].w += __uint_as_float(acc[q * 4 + 3]);
                m[q * 4 + 0] = v[q].x; m[q * 4 + 1] = v[q].y; m[q * 4 + 2] = v[q].z; m[q * 4 + 3] = v[q].w;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) o4[q] = v[q];
            if (p.x_out != nullptr)
                residual32(p, (int64_t)b * p.n + (int64_t)c * p.chunk + r, td * 128 + cc * 32, m);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<L::kTmemCols>(tmem);
    }
}

bool mlp_tc_supported(int64_t d, int64_t chunk) {
    return d % 128 == 0 && chunk >= 1 && chunk <= 256;
}

template <int NT>
static cudaError_t launch_smlp(const void* x, const void* w1, const float* b1, const void* w2,
                               const int32_t* idx, const int32_t* counts, int64_t k_max,
                               int64_t chunk, int64_t batch, int64_t n, int64_t d, int64_t f,
                               void* act_cm, float* out_cache, void* delta_ws, int64_t k_pad,
                               cudaStream_t s, const void* x_mid, void* x_out) {
    using L = MlpLayout<NT>;
    const int64_t nc = n / chunk;
    CUtensorMap tx, tw1, tdl, tw2;
    if (!make_map_bf16(&tx, x, d, batch * n, d, 128) || !make_map_bf16(&tw1, w1, d, f, d, 1) ||
        !make_map_bf16(&tdl, delta_ws, k_pad, batch * nc * chunk, k_pad, 128) ||
        !make_map_bf16(&tw2, w2, d, f, d, 1))
        return cudaErrorInvalidValue;
    MlpParams p{};
    p.idx = idx;
    p.counts = counts;
    p.k_max = (int)k_max;
    p.k_pad = (int)k_pad;
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
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_smlp_up<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemAlloc);
        cudaFuncSetAttribute(k_smlp_down<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemAlloc);
        attr = true;
    }
    dim3 g1((unsigned)((k_max + 127) / 128), (unsigned)(batch * nc));
    k_smlp_up<NT><<<g1, L::kThreads, L::kSmemAlloc, s>>>(tx, tw1, p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    dim3 g2((unsigned)(d / 128), (unsigned)(batch * nc));
    k_smlp_down<NT><<<g2, L::kThreads, L::kSmemAlloc, s>>>(tdl, tw2, p);
    return cudaGetLastError();
}

// delta workspace: [B*C*chunk rows][k_pad] bf16, k_pad = round_up(k_max, 128)
cudaError_t prod_sparse_delta_mlp_tc(const void* x, const void* w1, const float* b1,
                                     const void* w2, const int32_t* idx, const int32_t* counts,
                                     int64_t k_max, int64_t chunk, int64_t batch, int64_t n,
                                     int64_t d, int64_t f, void* act_cm, float* out_cache,
                                     void* delta_ws, cudaStream_t s, const void* x_mid,
                                     void* x_out) {
    if (!mlp_tc_supported(d, chunk)) return cudaErrorNotSupported;
    if (k_max == 0) return cudaSuccess;
    const int64_t k_pad = (k_max + 127) / 128 * 128;
    if (chunk > 128)
        return launch_smlp<2>(x, w1, b1, w2, idx, counts, k_max, chunk, batch, n, d, f, act_cm,
                              out_cache, delta_ws, k_pad, s, x_mid, x_out);
    return launch_smlp<1>(x, w1, b1, w2, idx, counts, k_max, chunk, batch, n, d, f, act_cm,
                          out_cache, delta_ws, k_pad, s, x_mid, x_out);
}

}  // namespace dev
}  // namespace csd
