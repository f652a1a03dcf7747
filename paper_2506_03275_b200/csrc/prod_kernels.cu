// prod_kernels.cu — CSD_MODE_PROD MLP-side kernels (bf16 storage, fp32 math).
//
//   tile means (mlp.cpp:83-96): chunk means of x, then T = means @ W1^T
//   casts, |delta| scores, bias/GELU epilogue of the dense (cuBLAS) MLP, and the
//   activation-cache layout conversions (reference [B,N,F] <-> chunk-major
//   [B,C,F,chunk] used by the tcgen05 sparse-delta MLP in mlp_tc.cu).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace csd {
namespace dev {

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

// chunk means of bf16 x -> fp32 [B*C, D]
__global__ void k_chunk_mean_bf16(const __nv_bfloat16* x, int64_t n, int64_t d, int64_t chunk,
                                  int64_t bc_total, float* out) {
    const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t bc = blockIdx.y;
    if (col >= d || bc >= bc_total) return;
    const int64_t nc = n / chunk;
    const int64_t b = bc / nc, c = bc % nc;
    const __nv_bfloat16* src = x + (b * n + c * chunk) * d + col;
    float s = 0.f;
    for (int64_t r = 0; r < chunk; ++r) s += __bfloat162float(src[r * d]);
    out[bc * d + col] = s * (1.0f / (float)chunk);
}

constexpr int GT = 64, GK = 32;

// T[bc, f] = means[bc, :] . W1[f, :]   grid (F/64, ceil(BC/64))
__global__ void __launch_bounds__(256)
k_means_w1(const float* __restrict__ means, const __nv_bfloat16* __restrict__ w1, int64_t bc,
           int64_t d, int64_t f, float* __restrict__ out) {
    __shared__ float As[GK][GT + 1];
    __shared__ float Bs[GK][GT + 1];
    const int64_t n0 = (int64_t)blockIdx.x * GT, m0 = (int64_t)blockIdx.y * GT;
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    float acc[4][4] = {};
    for (int64_t k0 = 0; k0 < d; k0 += GK) {
        for (int i = tid; i < GT * GK; i += 256) {
            const int r = i / GK, kk = i % GK;
            const int64_t gm = m0 + r, gn = n0 + r, gk = k0 + kk;
            As[kk][r] = (gm < bc && gk < d) ? means[gm * d + gk] : 0.f;
            Bs[kk][r] = (gn < f && gk < d) ? __bfloat162float(w1[gn * d + gk]) : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < GK; ++kk) {
            float av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) { av[i] = As[kk][ty * 4 + i]; bv[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) acc[i][jj] += av[i] * bv[jj];
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t r = m0 + ty * 4 + i;
        if (r >= bc) continue;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int64_t col = n0 + tx * 4 + jj;
            if (col < f) out[r * f + col] = acc[i][jj];
        }
    }
}

cudaError_t prod_tile_means(const void* x, const void* w1, int64_t batch, int64_t n, int64_t d,
                            int64_t f, int64_t chunk, float* means_ws, float* out,
                            cudaStream_t s) {
    const int64_t bc = batch * (n / chunk);
    dim3 g((unsigned)((d + 127) / 128), (unsigned)bc);
    k_chunk_mean_bf16<<<g, 128, 0, s>>>((const __nv_bfloat16*)x, n, d, chunk, bc, means_ws);
    dim3 g2((unsigned)((f + GT - 1) / GT), (unsigned)((bc + GT - 1) / GT));
    k_means_w1<<<g2, 256, 0, s>>>(means_ws, (const __nv_bfloat16*)w1, bc, d, f, out);
    return cudaGetLastError();
}

// act [B*N, F] bf16 (row-major, from the dense GEMM1) -> chunk-major cache
__global__ void k_act_to_cm(const __nv_bfloat16* act, int64_t n, int64_t f, int64_t chunk,
                            int64_t total_rows, __nv_bfloat16* cm) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total_rows * f) return;
    const int64_t row = i / f, col = i % f;      // row = b*n + tok
    const int64_t b = row / n, tok = row % n;
    const int64_t c = tok / chunk, r = tok % chunk;
    const int64_t nc = n / chunk;
    cm[(((b * nc + c) * f) + col) * chunk + r] = act[i];
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

// gelu + bias epilogue for the cuBLAS dense GEMM1: pre (fp32 [BN, F]) -> act bf16
__global__ void k_bias_gelu(const float* pre, const float* b1, int64_t rows, int64_t f,
                            __nv_bfloat16* act) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * f) return;
    act[i] = __float2bfloat16_rn(fast_gelu(pre[i] + b1[i % f]));
}
__global__ void k_bias_add_rows(float* out, const float* b2, int64_t rows, int64_t d) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < rows * d) out[i] += b2[i % d];
}

cudaError_t prod_bias_gelu(const float* pre, const float* b1, int64_t rows, int64_t f, void* act,
                           cudaStream_t s) {
    const int64_t t = rows * f;
    k_bias_gelu<<<(unsigned)((t + 255) / 256), 256, 0, s>>>(pre, b1, rows, f, (__nv_bfloat16*)act);
    return cudaGetLastError();
}
cudaError_t prod_bias_add_rows(float* out, const float* b2, int64_t rows, int64_t d,
                               cudaStream_t s) {
    const int64_t t = rows * d;
    k_bias_add_rows<<<(unsigned)((t + 255) / 256), 256, 0, s>>>(out, b2, rows, d);
    return cudaGetLastError();
}
cudaError_t prod_act_to_cm(const void* act, int64_t batch, int64_t n, int64_t f, int64_t chunk,
                           void* cm, cudaStream_t s) {
    const int64_t tot = batch * n * f;
    k_act_to_cm<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>((const __nv_bfloat16*)act, n, f,
                                                            chunk, batch * n, (__nv_bfloat16*)cm);
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
