// prod_kernels.cu — CSD_MODE_PROD MLP-side kernels (bf16 storage, fp32 math).
//
//   tile means (mlp.cpp:83-96): chunk means of x, then T = means @ W1^T
//   casts, |delta| scores, bias/GELU epilogue of the dense (cuBLAS) MLP, and the
//   activation-cache layout conversions (reference [B,N,F] <-> chunk-major
//   [B,C,F,chunk] used by the tcgen05 sparse-delta MLP in mlp_tc.cu).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "tc_common.cuh"
#include "kernels.h"

namespace csd {
namespace dev {
using csd::tc::pack_bf16x2;

__global__ void k_cast_f32_bf16(const float* in, __nv_bfloat16* out, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = __float2bfloat16_rn(in[i]);
}
__global__ void k_cast_bf16_f32(const __nv_bfloat16* in, float* out, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = __bfloat162float(in[i]);
}
cudaError_t prod_cast_f32_bf16(const float* in, void* out, int64_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_cast_f32_bf16<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, (__nv_bfloat16*)out, n);
    return cudaGetLastError();
}
cudaError_t prod_cast_bf16_f32(const void* in, float* out, int64_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_cast_bf16_f32<<<(unsigned)((n + 255) / 256), 256, 0, s>>>((const __nv_bfloat16*)in, out, n);
    return cudaGetLastError();
}

__global__ void k_absdiff_f(const float* a, const float* b, int64_t n, float* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = fabsf(a[i] - b[i]);
}
cudaError_t prod_absdiff(const float* a, const float* b, int64_t numel, float* out,
                         cudaStream_t s) {
    k_absdiff_f<<<(unsigned)((numel + 255) / 256), 256, 0, s>>>(a, b, numel, out);
    return cudaGetLastError();
}

// Dense-step MLP epilogue, fused (mlp.cpp:57-62 + cache refresh mlp.cpp:196-205):
// pre (bf16 [B*N, F], from the dense GEMM1) -> act = gelu(pre + b1) written row-major
// (GEMM2 operand) AND transposed into the chunk-major activation cache [B,C,F,chunk],
// through a 64x64 shared-memory tile so both writes are coalesced.
__global__ void __launch_bounds__(256)
k_bias_gelu_cm(const __nv_bfloat16* __restrict__ pre, const float* __restrict__ b1, int64_t n,
               int64_t f, int64_t chunk, __nv_bfloat16* __restrict__ act,
               __nv_bfloat16* __restrict__ cm) {
    // 16-byte accesses in both passes: row pass = 8 columns per thread-step, chunk-major
    // pass = 8 consecutive rows of one column per thread-step (tile pitch 72 bf16: the
    // column reads of the second pass hit distinct banks)
    __shared__ __align__(16) __nv_bfloat16 tile[64][72];
    const int64_t z = blockIdx.z;  // b * C + c
    const int64_t nc = n / chunk;
    const int64_t b = z / nc, c = z % nc;
    const int64_t r0 = (int64_t)blockIdx.y * 64, f0 = (int64_t)blockIdx.x * 64;
    const int tid = threadIdx.x;
    const int cg = tid & 7;  // 8-column group
    float bias[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) bias[u] = b1[f0 + cg * 8 + u];
#pragma unroll
    for (int rep = 0; rep < 2; ++rep) {
        const int rr = (tid >> 3) + rep * 32;
        const int64_t r = r0 + rr;
        if (r >= chunk) continue;
        const int64_t row = b * n + c * chunk + r;
        const uint4 pv = *reinterpret_cast<const uint4*>(pre + row * f + f0 + cg * 8);
        const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&pv);
        uint32_t o[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float2 pf = __bfloat1622float2(p2[u]);
            o[u] = pack_bf16x2(gelu_tanh_approx(pf.x + bias[2 * u]), gelu_tanh_approx(pf.y + bias[2 * u + 1]));
        }
        const uint4 ov = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4*>(act + row * f + f0 + cg * 8) = ov;
        *reinterpret_cast<uint4*>(&tile[rr][cg * 8]) = ov;
    }
    __syncthreads();
    // chunk-major pass: cm[z][f0 + j][r0 + 8 g .. + 7]
#pragma unroll
    for (int rep = 0; rep < 2; ++rep) {
        const int jj = (tid >> 3) + rep * 32, g8 = tid & 7;
        const int64_t rbase = r0 + g8 * 8;
        if (rbase >= chunk) continue;
        uint32_t w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const __nv_bfloat16 lo = tile[g8 * 8 + 2 * u][jj], hi = tile[g8 * 8 + 2 * u + 1][jj];
            w[u] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
        }
        __nv_bfloat16* dst = cm + (z * f + f0 + jj) * chunk + rbase;
        if (rbase + 8 <= chunk) {
            *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
            for (int i = 0; i < (int)(chunk - rbase); ++i) dst[i] = tile[g8 * 8 + i][jj];
        }
    }
}
// Same epilogue, one CTA per (chunk, 64 hidden columns) covering all `chunk` rows: warp w
// owns 8-column group w, lane l row pairs (2p, 2p+1), p = l + 32 * band.  All loads of the
// CTA are issued before any math; each row pair's 8 GELU'd columns are packed as words
// (row 2p | row 2p+1 << 16) into tile_t[col][p], so the chunk-major pass reads 16-byte runs
// of 8 rows of one column and the CTA's 64 x chunk output block — contiguous in the
// [B, C, F, chunk] cache — is written as one linear run of 16-byte stores.  `act` may be
// null: the dense GEMM2 then reads the chunk-major cache directly (prod_dense_mlp).
template <int kBands>  // ceil(chunk / 64)
__global__ void __launch_bounds__(256)
k_bias_gelu_cm_rows(const __nv_bfloat16* __restrict__ pre, const float* __restrict__ b1,
                    int64_t n, int64_t f, int64_t chunk, __nv_bfloat16* __restrict__ act,
                    __nv_bfloat16* __restrict__ cm) {
    extern __shared__ __align__(16) uint32_t tile_t[];  // [64][pw] words
    const int pw = (int)(chunk / 2) + 4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t z = blockIdx.y, nc = n / chunk;
    const int64_t b = z / nc, c = z % nc;
    const int64_t f0 = (int64_t)blockIdx.x * 64, col = f0 + warp * 8;
    const int64_t row0 = b * n + c * chunk;
    uint4 v[kBands][2];
#pragma unroll
    for (int band = 0; band < kBands; ++band) {
        const int64_t r = 2 * (lane + 32 * band);
        if (r < chunk) {
            v[band][0] = __ldg(reinterpret_cast<const uint4*>(pre + (row0 + r) * f + col));
            v[band][1] = __ldg(reinterpret_cast<const uint4*>(pre + (row0 + r + 1) * f + col));
        }
    }
    float bias[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) bias[u] = b1[col + u];
#pragma unroll
    for (int band = 0; band < kBands; ++band) {
        const int p = lane + 32 * band;
        const int64_t r = 2 * p;
        if (r >= chunk) continue;
        uint32_t o[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&v[band][h]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float2 pf = __bfloat1622float2(p2[u]);
                o[h][u] = pack_bf16x2(gelu_tanh_approx(pf.x + bias[2 * u]),
                                      gelu_tanh_approx(pf.y + bias[2 * u + 1]));
            }
            if (act != nullptr)
                *reinterpret_cast<uint4*>(act + (row0 + r + h) * f + col) =
                    make_uint4(o[h][0], o[h][1], o[h][2], o[h][3]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // columns 2u, 2u+1: interleave the two rows
            tile_t[(warp * 8 + 2 * u) * pw + p] = __byte_perm(o[0][u], o[1][u], 0x5410);
            tile_t[(warp * 8 + 2 * u + 1) * pw + p] = __byte_perm(o[0][u], o[1][u], 0x7632);
        }
    }
    __syncthreads();
    const int per_col = (int)(chunk / 8);  // 16-byte pieces per column
    uint4* dst = reinterpret_cast<uint4*>(cm + (z * f + f0) * chunk);
    for (int piece = threadIdx.x; piece < 64 * per_col; piece += 256) {
        const int jj = piece / per_col, q = piece - jj * per_col;
        dst[piece] = *reinterpret_cast<const uint4*>(tile_t + jj * pw + 4 * q);
    }
}

__global__ void k_cm_to_ref(const __nv_bfloat16* cm, int64_t n, int64_t f, int64_t chunk,
                            int64_t total_rows, float* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total_rows * f) return;
    const int64_t row = i / f, col = i % f;
    const int64_t b = row / n, tok = row % n;
    const int64_t c = tok / chunk, r = tok % chunk;
    const int64_t nc = n / chunk;
    out[i] = __bfloat162float(cm[(((b * nc + c) * f) + col) * chunk + r]);
}
cudaError_t prod_act_cm_to_ref(const void* act_cm, int64_t batch, int64_t n, int64_t f,
                               int64_t chunk, float* out, cudaStream_t s) {
    const int64_t tot = batch * n * f;
    k_cm_to_ref<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>((const __nv_bfloat16*)act_cm, n, f,
                                                            chunk, batch * n, out);
    return cudaGetLastError();
}

// out (fp32 M_cache) += b2 per row; optionally x_out = bf16(x_mid + out) in the same pass.
// grid (d / 4 / 256 rounded up, rows); 4 columns per thread (float4 / 8-byte bf16 accesses).
__global__ void k_bias_add_rows(float* __restrict__ out, const float* __restrict__ b2, int64_t d,
                                const __nv_bfloat16* __restrict__ x_mid,
                                __nv_bfloat16* __restrict__ x_out) {
    const int64_t row = blockIdx.y;
    const int col = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (col >= d) return;
    float4* o4 = reinterpret_cast<float4*>(out + row * d + col);
    const float4 bb = *reinterpret_cast<const float4*>(b2 + col);
    float4 v = *o4;
    v.x += bb.x; v.y += bb.y; v.z += bb.z; v.w += bb.w;
    *o4 = v;
    if (x_out) {
        const uint2 xr = *reinterpret_cast<const uint2*>(x_mid + row * d + col);
        const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&xr);
        const float2 a = __bfloat1622float2(xh[0]), b = __bfloat1622float2(xh[1]);
        uint2 w;
        __nv_bfloat162 r0 = __floats2bfloat162_rn(a.x + v.x, a.y + v.y);
        __nv_bfloat162 r1 = __floats2bfloat162_rn(b.x + v.z, b.y + v.w);
        w.x = *reinterpret_cast<uint32_t*>(&r0);
        w.y = *reinterpret_cast<uint32_t*>(&r1);
        *reinterpret_cast<uint2*>(x_out + row * d + col) = w;
    }
}

cudaError_t prod_bias_gelu_cm(const void* pre, const float* b1, int64_t batch, int64_t n,
                              int64_t f, int64_t chunk, void* act, void* cm, cudaStream_t s) {
    if (f % 64 || chunk % 8) return cudaErrorNotSupported;  // 16-byte chunk-major rows
    if (chunk <= 256) {
        const dim3 gr((unsigned)(f / 64), (unsigned)(batch * (n / chunk)));
        const size_t sm = 64 * (size_t)(chunk / 2 + 4) * 4;
        const auto* pp = (const __nv_bfloat16*)pre;
        auto* a = (__nv_bfloat16*)act;
        auto* m = (__nv_bfloat16*)cm;
        const int bands = (int)((chunk + 63) / 64);
        if (bands == 1) k_bias_gelu_cm_rows<1><<<gr, 256, sm, s>>>(pp, b1, n, f, chunk, a, m);
        else if (bands == 2) k_bias_gelu_cm_rows<2><<<gr, 256, sm, s>>>(pp, b1, n, f, chunk, a, m);
        else if (bands == 3) k_bias_gelu_cm_rows<3><<<gr, 256, sm, s>>>(pp, b1, n, f, chunk, a, m);
        else k_bias_gelu_cm_rows<4><<<gr, 256, sm, s>>>(pp, b1, n, f, chunk, a, m);
        return cudaGetLastError();
    }
    dim3 g((unsigned)(f / 64), (unsigned)((chunk + 63) / 64), (unsigned)(batch * (n / chunk)));
    k_bias_gelu_cm<<<g, 256, 0, s>>>((const __nv_bfloat16*)pre, b1, n, f, chunk,
                                     (__nv_bfloat16*)act, (__nv_bfloat16*)cm);
    return cudaGetLastError();
}
cudaError_t prod_bias_add_rows(float* out, const float* b2, int64_t rows, int64_t d,
                               const void* x_mid, void* x_out, cudaStream_t s) {
    if (d % 4) return cudaErrorNotSupported;
    dim3 g((unsigned)((d / 4 + 255) / 256), (unsigned)rows);
    k_bias_add_rows<<<g, 256, 0, s>>>(out, b2, d, (const __nv_bfloat16*)x_mid,
                                      (__nv_bfloat16*)x_out);
    return cudaGetLastError();
}

}  // namespace dev
}  // namespace csd

namespace csd {
namespace dev {
__global__ void k_add_bf16_f32(const __nv_bfloat16* a, const float* b, int64_t n,
                               __nv_bfloat16* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = __float2bfloat16_rn(__bfloat162float(a[i]) + b[i]);
}
cudaError_t prod_add_bf16_f32(const void* a, const float* b, int64_t numel, void* out,
                              cudaStream_t s) {
    k_add_bf16_f32<<<(unsigned)((numel + 255) / 256), 256, 0, s>>>(
        (const __nv_bfloat16*)a, b, numel, (__nv_bfloat16*)out);
    return cudaGetLastError();
}
}  // namespace dev
}  // namespace csd
