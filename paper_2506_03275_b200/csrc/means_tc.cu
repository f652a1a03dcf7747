// means_tc.cu — MLP change-detection GEMM on tcgen05 (CSD_MODE_PROD).
//
// mlp_tile_means (mlp.cpp:83-96): T[bc, f] = chunk_mean(x)[bc, :] . W1[f, :]
// is a skinny GEMM (B*C = 24 chunk rows at FLUX) that must stream all of W1
// (F x D bf16 = 75.5 MB) — HBM-bound.  Layout for the tensor cores:
//   A = W1 rows (M = 128 neurons per tile, K-major, plain TMA tiles, no gather);
//   B = chunk means split into bf16 hi + lo parts (mean = hi + lo to ~2^-16 rel.),
//       tiles of cb <= 64 chunks laid out [cb hi rows | cb lo rows | zero pad to N],
//       N = round_up(2 cb, 16) (FLUX: 48), so T = acc[:, j] + acc[:, cb + j] keeps
//       fp32-grade precision for the |T - T_m| ranking;
//   split-K over the CTA grid (>= 148 CTAs) into per-split partial buffers that a
//   fixed-order reduction sums (deterministic — the top-k depends on it).
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

constexpr int kMeansStages = 4;
constexpr uint32_t kMTile = 128 * 128;  // 128 rows x 64 bf16

// tile of cb <= 64 chunks: hi rows [0, cb), lo rows [hipad, hipad + cb) with hipad =
// round_up(cb, 32) (32-aligned TMEM column groups in the epilogue); the gap / tail rows are
// never written and their accumulator columns are never read.
__host__ __device__ inline int means_tile_chunks(int bc_total, int nt) { return min(64, bc_total - nt * 64); }
__host__ __device__ inline int means_tile_hipad(int cb) { return (cb + 31) / 32 * 32; }
__host__ __device__ inline int means_tile_n(int cb) { return (means_tile_hipad(cb) + cb + 15) / 16 * 16; }

// x [B,N,D] bf16 -> B operand rows (hi/lo split): chunk bc -> tile t = bc / 64, j = bc % 64,
// hi row t*128 + j, lo row t*128 + hipad + j (see means_tile_hipad).  Block: 256 columns (lane = 8 columns, 16-byte loads), 8 warps split
// the chunk's rows, fixed-order smem reduction.
constexpr int kCmThreads = 256;
__global__ void __launch_bounds__(kCmThreads)
k_chunk_means_split(const __nv_bfloat16* __restrict__ x, int64_t n, int64_t d, int64_t chunk,
                    int64_t bc_total, __nv_bfloat16* __restrict__ bop) {
    __shared__ float part[8][256];
    pdl_wait();
    if (threadIdx.x == 0) pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t bc = blockIdx.y;
    const int64_t col0 = (int64_t)blockIdx.x * 256 + lane * 8;
    const int64_t nc = n / chunk;
    const int64_t b = bc / nc, c = bc % nc;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (col0 < d) {
        const __nv_bfloat16* src = x + (b * n + c * chunk) * d + col0;
#pragma unroll 24
        for (int64_t r = warp; r < chunk; r += 8) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + r * d));
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float2 f = __bfloat1622float2(h[u]);
                acc[2 * u] += f.x;
                acc[2 * u + 1] += f.y;
            }
        }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) part[warp][lane * 8 + u] = acc[u];
    __syncthreads();
    const int cl = threadIdx.x;  // column within the block
    const int64_t col = (int64_t)blockIdx.x * 256 + cl;
    if (col >= d) return;
    float sum = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) sum += part[w][cl];
    const float mean = sum * (1.0f / (float)chunk);
    const __nv_bfloat16 hi = __float2bfloat16_rn(mean);
    const __nv_bfloat16 lo = __float2bfloat16_rn(mean - __bfloat162float(hi));
    const int64_t t = bc / 64, j = bc % 64;
    const int cb = means_tile_chunks((int)bc_total, (int)t);
    bop[(t * 128 + j) * d + col] = hi;
    bop[(t * 128 + means_tile_hipad(cb) + j) * d + col] = lo;
}

struct MeansParams {
    float* partial;  // [ksplit][bc_total][f]
    int bc_total, f, kb_per_split;
    uint32_t b_slot;  // bytes per B stage slot (widest tile rows x 128 B)
};

__global__ void __launch_bounds__(128, 2)
k_tile_means_tc(const __grid_constant__ CUtensorMap tm_w1, const __grid_constant__ CUtensorMap tm_b,
                const MeansParams p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = blockIdx.x, nt = blockIdx.y, ks = blockIdx.z;
    const int kb0 = ks * p.kb_per_split;
    const int cb = means_tile_chunks(p.bc_total, nt), nrows = means_tile_n(cb);
    const uint32_t b_bytes = (uint32_t)nrows * 128u;  // B tile: nrows x 64 columns
    uint8_t* sA = smem;
    uint8_t* sB = smem + kMeansStages * kMTile;  // [stage] slots of p.b_slot bytes
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kMeansStages * (kMTile + p.b_slot));
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
    pdl_wait();
    if (threadIdx.x == 0) pdl_trigger();

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_w1);
        tma_prefetch_desc(&tm_b);
        for (int i = 0; i < p.kb_per_split; ++i) {
            const int s = i % kMeansStages;
            if (i >= kMeansStages) mbar_wait(empty + s, ((i / kMeansStages) - 1) & 1);
            mbar_arrive_expect_tx(full + s, kMTile + b_bytes);
            tma_load_2d(&tm_w1, full + s, sA + s * kMTile, (kb0 + i) * 64, mt * 128);
            for (int r16 = 0; r16 < nrows; r16 += 16)  // B: 16-row boxes, only the live rows
                tma_load_2d(&tm_b, full + s, sB + s * p.b_slot + r16 * 128, (kb0 + i) * 64, nt * 128 + r16);
        }
    } else if (warp == 1 && lane == 0) {
        const uint32_t id = idesc_bf16(128, (uint32_t)nrows, false, false);
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        for (int i = 0; i < p.kb_per_split; ++i) {
            const int s = i % kMeansStages;
            mbar_wait(full + s, (i / kMeansStages) & 1);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                mma_bf16(tmem, desc_kmajor_sw128(a0 + s * kMTile + kk * 32),
                         desc_kmajor_sw128(b0 + s * p.b_slot + kk * 32), id, (i > 0 || kk > 0) ? 1u : 0u);
            mma_commit(empty + s);
        }
        mma_commit(done);
    }
    __syncwarp();
    // epilogue: all 4 warps; thread = neuron row (TMEM lane)
    mbar_wait(done, 0);
    tc_fence_after();
    const uint32_t tacc = tmem + ((uint32_t)(warp * 32) << 16);
    const int f = mt * 128 + warp * 32 + lane;
    float* out = p.partial + (int64_t)ks * p.bc_total * p.f;
    // T[j] = acc[:, j] (hi) + acc[:, hipad + j] (lo), in 32-column groups
    const int hipad = means_tile_hipad(cb);
#pragma unroll 1
    for (int g = 0; g * 32 < cb; ++g) {
        uint32_t hv[32], lv[32];
        tmem_ld32(tacc + g * 32, hv);
        tmem_ld32(tacc + hipad + g * 32, lv);
        tmem_ld_wait();
        if (f < p.f) {
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
                const int j = g * 32 + jj;
                if (j < cb)
                    out[(int64_t)(nt * 64 + j) * p.f + f] = __uint_as_float(hv[jj]) + __uint_as_float(lv[jj]);
            }
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
    pdl_wait();
    if (threadIdx.x == 0) pdl_trigger();
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
                               float* out, void* ws, cudaStream_t s, MeansPartials* partials_out) {
    if (d % 64 || f % 128) return cudaErrorNotSupported;
    const int64_t bc = batch * (n / chunk);
    const int64_t ntiles = (bc + 63) / 64;
    const int64_t mtiles = f / 128, kblocks = d / 64;
    const int ks = pick_ksplit(mtiles * ntiles, kblocks);
    __nv_bfloat16* bop = (__nv_bfloat16*)ws;
    float* partial = (float*)((char*)ws + ((2 * ntiles * 128 * d + 255) / 256) * 256);
    dim3 g1((unsigned)((d + 255) / 256), (unsigned)bc);
    {
        cudaError_t e = launch_ex(k_chunk_means_split, g1, dim3(kCmThreads), 0, s, 1,
                                  (const __nv_bfloat16*)x, n, d, chunk, bc, bop);
        if (e != cudaSuccess) return e;
    }
    CUtensorMap tw, tb;
    if (!make_map_bf16(&tw, w1, d, f, d, 128) || !make_map_bf16(&tb, bop, d, ntiles * 128, d, 16))
        return cudaErrorInvalidValue;
    // B slots sized for the widest tile: 2 CTAs per SM when the B tiles are narrow
    const int nmax = means_tile_n(means_tile_chunks((int)bc, 0));
    MeansParams p{partial, (int)bc, (int)f, (int)(kblocks / ks), (uint32_t)nmax * 128u};
    const size_t smem = kMeansStages * (kMTile + (size_t)nmax * 128) + 256 + 1024;
    {
        cudaError_t e = ensure_smem_attr(k_tile_means_tc, 227 * 1024);
        if (e != cudaSuccess) return e;
    }
    {
        cudaError_t e = launch_ex(k_tile_means_tc, dim3((unsigned)mtiles, (unsigned)ntiles, (unsigned)ks),
                                  dim3(128), smem, s, 1, tw, tb, p);
        if (e != cudaSuccess) return e;
    }
    const int64_t total = bc * f;
    if (partials_out != nullptr) {  // the caller fuses the reduction (top-k load)
        partials_out->partial = partial;
        partials_out->ks = ks;
        return cudaGetLastError();
    }
    return launch_ex(k_means_reduce, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, s, 1,
                     (const float*)partial, ks, total, cached, out);
}

size_t prod_means_ws_bytes(int64_t batch, int64_t n, int64_t d, int64_t f, int64_t chunk) {
    const int64_t bc = batch * (n / chunk);
    const int64_t ntiles = (bc + 63) / 64;
    return ((2 * ntiles * 128 * d + 255) / 256) * 256 + 4 * 8 * bc * f;
}

bool means_tc_supported(int64_t d, int64_t f) { return d % 64 == 0 && f % 128 == 0; }

}  // namespace dev
}  // namespace csd
