// means_tc.cu — MLP change-detection GEMM on tcgen05 (CSD_MODE_PROD).
//
// mlp_tile_means (mlp.cpp:83-96): T[bc, f] = chunk_mean(x)[bc, :] . W1[f, :]
// is a skinny GEMM (B*C = 24 chunk rows at FLUX) that must stream all of W1
// (F x D bf16 = 75.5 MB) — HBM-bound.  Layout for the tensor cores:
//   A = W1 rows (M = 128 neurons per tile, K-major, plain TMA tiles, no gather);
//   B = chunk means split into bf16 hi + lo parts (mean = hi + lo to ~2^-16 rel.),
//       128-row tiles [64 hi rows | 64 lo rows], so T = acc[:, j] + acc[:, 64 + j]
//       keeps fp32-grade precision for the |T - T_m| ranking;
//   split-K over the CTA grid (>= 148 CTAs) into per-split partial buffers that a
//   fixed-order reduction sums (deterministic — the top-k depends on it).
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

constexpr int kMeansStages = 4;
constexpr uint32_t kMTile = 128 * 128;  // 128 rows x 64 bf16

// x [B,N,D] bf16 -> B operand [ntiles*128, D] bf16 (hi/lo split), chunk bc -> tile bc/64
__global__ void k_chunk_means_split(const __nv_bfloat16* __restrict__ x, int64_t n, int64_t d,
                                    int64_t chunk, int64_t bc_total,
                                    __nv_bfloat16* __restrict__ bop) {
    const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t bc = blockIdx.y;
    if (col >= d || bc >= bc_total) return;
    const int64_t nc = n / chunk;
    const int64_t b = bc / nc, c = bc % nc;
    const __nv_bfloat16* src = x + (b * n + c * chunk) * d + col;
    float s = 0.f;
#pragma unroll 16
    for (int64_t r = 0; r < chunk; ++r) s += __bfloat162float(__ldg(src + r * d));
    const float mean = s * (1.0f / (float)chunk);
    const __nv_bfloat16 hi = __float2bfloat16_rn(mean);
    const __nv_bfloat16 lo = __float2bfloat16_rn(mean - __bfloat162float(hi));
    const int64_t t = bc / 64, j = bc % 64;
    bop[(t * 128 + j) * d + col] = hi;
    bop[(t * 128 + 64 + j) * d + col] = lo;
}

struct MeansParams {
    float* partial;  // [ksplit][bc_total][f]
    int bc_total, f, kb_per_split;
};

__global__ void __launch_bounds__(128, 1)
k_tile_means_tc(const __grid_constant__ CUtensorMap tm_w1, const __grid_constant__ CUtensorMap tm_b,
                const MeansParams p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = blockIdx.x, nt = blockIdx.y, ks = blockIdx.z;
    const int kb0 = ks * p.kb_per_split;
    uint8_t* sA = smem;
    uint8_t* sB = smem + kMeansStages * kMTile;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kMeansStages * kMTile);
    uint64_t* full = bars;
    uint64_t* empty = bars + kMeansStages;
    uint64_t* done = bars + 2 * kMeansStages;
    uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 2 * kMeansStages + 1);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kMeansStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        mbar_init(done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<128>(slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_w1);
        tma_prefetch_desc(&tm_b);
        for (int i = 0; i < p.kb_per_split; ++i) {
            const int s = i % kMeansStages;
            if (i >= kMeansStages) mbar_wait(empty + s, ((i / kMeansStages) - 1) & 1);
            mbar_arrive_expect_tx(full + s, 2 * kMTile);
            tma_load_2d(&tm_w1, full + s, sA + s * kMTile, (kb0 + i) * 64, mt * 128);
            tma_load_2d(&tm_b, full + s, sB + s * kMTile, (kb0 + i) * 64, nt * 128);
        }
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t id = idesc_bf16(128, 128, false, false);
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        for (int i = 0; i < p.kb_per_split; ++i) {
            const int s = i % kMeansStages;
            mbar_wait(full + s, (i / kMeansStages) & 1);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                mma_bf16(tmem, desc_kmajor_sw128(a0 + s * kMTile + kk * 32),
                         desc_kmajor_sw128(b0 + s * kMTile + kk * 32), id, (i > 0 || kk > 0) ? 1u : 0u);
            mma_commit(empty + s);
        }
        mma_commit(done);
    }
    __syncwarp();
    // epilogue: all 4 warps; thread = neuron row (TMEM lane)
    mbar_wait(done, 0);
    tc_fence_after();
    const uint32_t tacc = tmem + ((uint32_t)(warp * 32) << 16);
    uint32_t hi[32], lo[32];
    const int f = mt * 128 + warp * 32 + lane;
    float* out = p.partial + (int64_t)ks * p.bc_total * p.f;
#pragma unroll 1
    for (int cc = 0; cc < 2; ++cc) {
        tmem_ld32(tacc + cc * 32, hi);
        tmem_ld32(tacc + 64 + cc * 32, lo);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int bc = nt * 64 + cc * 32 + j;
            if (bc < p.bc_total && f < p.f)
                out[(int64_t)bc * p.f + f] = __uint_as_float(hi[j]) + __uint_as_float(lo[j]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<128>(tmem);
    }
}

// out = sum_k partial[k] (fixed order); with `cached`: out = |sum - cached| (mlp.cpp:116)
__global__ void k_means_reduce(const float* __restrict__ partial, int ksplit, int64_t total,
                               const float* __restrict__ cached, float* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    float s = partial[i];
    for (int k = 1; k < ksplit; ++k) s += partial[(int64_t)k * total + i];
    out[i] = cached ? fabsf(s - cached[i]) : s;
}

// The split depends on D only — never on the neuron count — so a hidden-column shard
// (F/g neurons on each of g GPUs) produces bit-identical T values and therefore the same
// global top-k as one GPU.
static int pick_ksplit(int64_t /*tiles*/, int64_t kblocks) { return kblocks % 2 == 0 ? 2 : 1; }

// T (or |T - cached| when cached != null) for the chunk means of x.
// ws: bop [ntiles*128, D] bf16 + partials [ksplit][BC][F] fp32 (see prod_means_ws_bytes).
cudaError_t prod_tile_means_tc(const void* x, const void* w1, int64_t batch, int64_t n,
                               int64_t d, int64_t f, int64_t chunk, const float* cached,
                               float* out, void* ws, cudaStream_t s) {
    if (d % 64 || f % 128) return cudaErrorNotSupported;
    const int64_t bc = batch * (n / chunk);
    const int64_t ntiles = (bc + 63) / 64;
    const int64_t mtiles = f / 128, kblocks = d / 64;
    const int ks = pick_ksplit(mtiles * ntiles, kblocks);
    __nv_bfloat16* bop = (__nv_bfloat16*)ws;
    float* partial = (float*)((char*)ws + ((2 * ntiles * 128 * d + 255) / 256) * 256);
    cudaError_t e = cudaMemsetAsync(bop, 0, 2 * ntiles * 128 * d, s);
    if (e != cudaSuccess) return e;
    dim3 g1((unsigned)((d + 127) / 128), (unsigned)bc);
    k_chunk_means_split<<<g1, 128, 0, s>>>((const __nv_bfloat16*)x, n, d, chunk, bc, bop);
    CUtensorMap tw, tb;
    if (!make_map_bf16(&tw, w1, d, f, d, 128) || !make_map_bf16(&tb, bop, d, ntiles * 128, d, 128))
        return cudaErrorInvalidValue;
    MeansParams p{partial, (int)bc, (int)f, (int)(kblocks / ks)};
    const size_t smem = 2 * kMeansStages * kMTile + 256 + 1024;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_tile_means_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    k_tile_means_tc<<<dim3((unsigned)mtiles, (unsigned)ntiles, (unsigned)ks), 128, smem, s>>>(tw, tb, p);
    const int64_t total = bc * f;
    k_means_reduce<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(partial, ks, total, cached, out);
    return cudaGetLastError();
}

size_t prod_means_ws_bytes(int64_t batch, int64_t n, int64_t d, int64_t f, int64_t chunk) {
    const int64_t bc = batch * (n / chunk);
    const int64_t ntiles = (bc + 63) / 64;
    return ((2 * ntiles * 128 * d + 255) / 256) * 256 + 4 * 8 * bc * f;
}

bool means_tc_supported(int64_t d, int64_t f) { return d % 64 == 0 && f % 128 == 0; }

}  // namespace dev
}  // namespace csd
