// generation.cu — the multi-step schedule driver's device pieces.
//
//   csd_resolve_schedule    : dense / sparse / skipped plan (schedule.cpp:44-87, :21-41)
//   csd_latent_axpy         : latent += a * model_output (harness.cpp:24-30, used at :200)
//   csd_r_squared           : R^2 of (truth - origin) vs (approx - origin) in double
//                             (metrics.cpp:5-30 over harness.cpp:32-38 deltas)
//   csd_index_set_to_masks  : bitpacked per-chunk masks of an index set (bitmask.cpp:55-85)
//
// The latent is an fp32 master in both modes (the reference keeps fp32); in PROD the block
// output is bf16 and the axpy also refreshes a bf16 shadow copy that feeds the next step's
// blocks.  Compiled with -fmad=false (build.py) so the CHECK axpy is the reference's
// separate multiply and add.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "capi_internal.h"

namespace csd {
namespace dev {

// CHECK: o[i] += a * y[i] with fp32 y (harness.cpp:28; no contraction in this file)
__global__ void k_axpy_f32(float* __restrict__ latent, float a, const float* __restrict__ y,
                           int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) latent[i] = latent[i] + a * y[i];
}

// PROD: 8 elements per thread, bf16 y, fp32 master, optional bf16 shadow of the result
__global__ void k_axpy_bf16(float* __restrict__ latent, float a,
                            const __nv_bfloat16* __restrict__ y, int64_t n,
                            __nv_bfloat16* __restrict__ shadow) {
    const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (i0 >= n) return;
    if (i0 + 8 <= n) {
        float4 l0 = *reinterpret_cast<const float4*>(latent + i0);
        float4 l1 = *reinterpret_cast<const float4*>(latent + i0 + 4);
        const uint4 yv = *reinterpret_cast<const uint4*>(y + i0);
        const __nv_bfloat162* y2 = reinterpret_cast<const __nv_bfloat162*>(&yv);
        float2 f;
        f = __bfloat1622float2(y2[0]); l0.x = l0.x + a * f.x; l0.y = l0.y + a * f.y;
        f = __bfloat1622float2(y2[1]); l0.z = l0.z + a * f.x; l0.w = l0.w + a * f.y;
        f = __bfloat1622float2(y2[2]); l1.x = l1.x + a * f.x; l1.y = l1.y + a * f.y;
        f = __bfloat1622float2(y2[3]); l1.z = l1.z + a * f.x; l1.w = l1.w + a * f.y;
        *reinterpret_cast<float4*>(latent + i0) = l0;
        *reinterpret_cast<float4*>(latent + i0 + 4) = l1;
        if (shadow != nullptr) {
            __nv_bfloat162 s[4] = {__floats2bfloat162_rn(l0.x, l0.y), __floats2bfloat162_rn(l0.z, l0.w),
                                   __floats2bfloat162_rn(l1.x, l1.y), __floats2bfloat162_rn(l1.z, l1.w)};
            *reinterpret_cast<uint4*>(shadow + i0) = *reinterpret_cast<const uint4*>(s);
        }
        return;
    }
    for (int64_t i = i0; i < n; ++i) {
        const float l = latent[i] + a * __bfloat162float(y[i]);
        latent[i] = l;
        if (shadow != nullptr) shadow[i] = __float2bfloat16_rn(l);
    }
}

constexpr int kR2Blocks = 296;  // 2 x 148 SMs
constexpr int kR2Threads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];  // fixed order
    return s;
}

// pass 0: partial sums of d = t - o; pass 1: partial ss_res = sum (d_t - d_a)^2 and
// ss_tot = sum (d_t - mean)^2, mean = ws[0] / n (written by k_r2_final pass 0).
// Deterministic: fixed grid, grid-stride ranges, fixed-order block and final reductions.
__global__ void __launch_bounds__(kR2Threads)
k_r2_partial(const float* __restrict__ t, const float* __restrict__ a,
             const float* __restrict__ o, int64_t n, int pass, double* __restrict__ ws) {
    __shared__ double sh[kR2Threads / 32];
    const double mean = pass == 1 ? ws[0] / (double)n : 0.0;
    double s0 = 0.0, s1 = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double org = o != nullptr ? (double)o[i] : 0.0;
        const double dt = (double)t[i] - org;
        if (pass == 0) {
            s0 += dt;
        } else {
            const double da = (double)a[i] - org;
            s0 += (dt - da) * (dt - da);
            s1 += (dt - mean) * (dt - mean);
        }
    }
    const double r0 = block_sum(s0, sh);
    const double r1 = pass == 1 ? block_sum(s1, sh) : 0.0;
    if (threadIdx.x == 0) {
        ws[2 + 2 * blockIdx.x] = r0;
        ws[3 + 2 * blockIdx.x] = r1;
    }
}

// pass 0: ws[0] = sum; pass 1: ws[1] = 1 - ss_res / ss_tot (NaN when ss_tot == 0)
__global__ void k_r2_final(int pass, int nblocks, double* ws) {
    if (threadIdx.x != 0) return;
    double s0 = 0.0, s1 = 0.0;
    for (int b = 0; b < nblocks; ++b) {
        s0 += ws[2 + 2 * b];
        s1 += ws[3 + 2 * b];
    }
    if (pass == 0) ws[0] = s0;
    else ws[1] = s1 == 0.0 ? __longlong_as_double(0x7ff8000000000000ll) : 1.0 - s0 / s1;
}

// One CTA per (b, h, chunk) row: the row's n-bit mask is built in shared memory (32-bit
// words, atomicOr), checked (popcount == count, else a duplicate; ids in [0, n)), and
// written out as ceil(n / 8) bytes, LSB-first (bitmask.hpp:13-17) -- byte j of a
// little-endian word w is bits [8 j, 8 j + 8) of it.
__global__ void k_index_masks(const int32_t* __restrict__ idx, const int32_t* __restrict__ counts,
                              int64_t k_max, int64_t n, int64_t row_bytes,
                              uint8_t* __restrict__ masks, uint32_t* __restrict__ flags) {
    extern __shared__ uint32_t bits[];
    const int64_t row = blockIdx.x;
    const int64_t nw = (n + 31) / 32;
    for (int64_t w = threadIdx.x; w < nw; w += blockDim.x) bits[w] = 0u;
    __syncthreads();
    const int cnt = counts[row];
    if (cnt < 0 || cnt > k_max) {
        if (threadIdx.x == 0) atomicOr(flags, kFlagCountRange);
        return;
    }
    const int32_t* ids = idx + row * k_max;
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
        const int32_t id = ids[j];
        if (id < 0 || id >= n) {
            atomicOr(flags, kFlagIndexRange);
            continue;
        }
        atomicOr(&bits[id >> 5], 1u << (id & 31));
    }
    __syncthreads();
    int pc = 0;
    for (int64_t w = threadIdx.x; w < nw; w += blockDim.x) pc += __popc(bits[w]);
    for (int o = 16; o > 0; o >>= 1) pc += __shfl_xor_sync(0xffffffffu, pc, o);
    __shared__ int warp_pc[32];
    if ((threadIdx.x & 31) == 0) warp_pc[threadIdx.x >> 5] = pc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += warp_pc[w];
        if (tot != cnt) atomicOr(flags, kFlagIndexDup);  // (out-of-range ids already flagged)
    }
    const uint8_t* b8 = reinterpret_cast<const uint8_t*>(bits);
    uint8_t* dst = masks + row * row_bytes;
    for (int64_t j = threadIdx.x; j < row_bytes; j += blockDim.x) dst[j] = b8[j];
}

}  // namespace dev
}  // namespace csd

using csd::set_error;

#define CSD_CU_(expr)                                                         \
    do {                                                                      \
        const cudaError_t e_ = (expr);                                        \
        if (e_ != cudaSuccess) return csd::cuda_status(e_, "generation.cu"); \
    } while (0)

extern "C" {

csd_status csd_resolve_schedule(int64_t total_steps, int64_t dense_interval, int use_step_cache,
                                int64_t window, int64_t stride, int32_t* modes) {
    if (total_steps < 1)
        return set_error(CSD_ERR_CONFIG, "total_steps must be >= 1, got %lld", (long long)total_steps);
    if (dense_interval < 0)
        return set_error(CSD_ERR_CONFIG, "dense_interval must be >= 0, got %lld",
                         (long long)dense_interval);
    if (use_step_cache) {
        if (window < 1 || window > total_steps)
            return set_error(CSD_ERR_CONFIG, "step-cache window %lld outside [1, total_steps=%lld]",
                             (long long)window, (long long)total_steps);
        if (stride < 1)
            return set_error(CSD_ERR_CONFIG, "step-cache stride must be >= 1, got %lld",
                             (long long)stride);
    }
    if (modes == nullptr) return set_error(CSD_ERR_VALUE, "null modes buffer");
    // a dense refresh at every (dense_interval + 1) boundary, sparse in between
    for (int64_t s = 0; s < total_steps; ++s)
        modes[s] = (s % (dense_interval + 1) == 0) ? CSD_STEP_DENSE : CSD_STEP_SPARSE;
    if (use_step_cache) {
        // centred window; steps off the stride grid are skipped, step 0 never is
        const int64_t start = (total_steps - window) / 2;
        for (int64_t s = start; s < start + window; ++s)
            if (s != 0 && (s - start) % stride != 0) modes[s] = CSD_STEP_SKIPPED;
    }
    // the plan's invariants (schedule.cpp:21-41): opens dense, no sparse step without an
    // earlier dense one (a skipped window may swallow a dense boundary)
    bool have_dense = false;
    for (int64_t s = 0; s < total_steps; ++s) {
        if (modes[s] == CSD_STEP_DENSE) have_dense = true;
        if (modes[s] == CSD_STEP_SPARSE && !have_dense)
            return set_error(CSD_ERR_CONFIG, "sparse step %lld has no preceding dense step",
                             (long long)s);
    }
    if (modes[0] != CSD_STEP_DENSE) return set_error(CSD_ERR_CONFIG, "schedule must start dense");
    return CSD_OK;
}

csd_status csd_latent_axpy(csd_ctx* ctx, csd_mode mode, float* latent, float a, const void* y,
                           int64_t numel, void* latent_bf16, void* stream) {
    if (!ctx) return set_error(CSD_ERR_VALUE, "null context");
    if (numel < 0) return set_error(CSD_ERR_SHAPE, "negative element count");
    if (numel == 0) return CSD_OK;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (mode == CSD_MODE_PROD) {
        const int64_t th = (numel + 7) / 8;
        csd::dev::k_axpy_bf16<<<(unsigned)((th + 255) / 256), 256, 0, s>>>(
            latent, a, static_cast<const __nv_bfloat16*>(y), numel,
            static_cast<__nv_bfloat16*>(latent_bf16));
    } else {
        csd::dev::k_axpy_f32<<<(unsigned)((numel + 255) / 256), 256, 0, s>>>(
            latent, a, static_cast<const float*>(y), numel);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return csd::cuda_status(e, "latent_axpy");
    reinterpret_cast<csd::Ctx*>(ctx)->launches += 1;
    return CSD_OK;
}

csd_status csd_r_squared(csd_ctx* ctx, const float* truth, const float* approx,
                         const float* origin, int64_t numel, double* r2, void* stream) {
    if (!ctx) return set_error(CSD_ERR_VALUE, "null context");
    if (numel < 1) return set_error(CSD_ERR_SHAPE, "r_squared needs at least one element");
    if (!truth || !approx || !r2) return set_error(CSD_ERR_VALUE, "null r_squared argument");
    auto* c = reinterpret_cast<csd::Ctx*>(ctx);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    using namespace csd::dev;
    auto* ws = static_cast<double*>(c->ws(csd::kWsR2, sizeof(double) * (2 + 2 * kR2Blocks)));
    if (!ws) return set_error(CSD_ERR_CUDA, "workspace allocation failed");
    const int nb = (int)std::min<int64_t>(kR2Blocks, (numel + kR2Threads - 1) / kR2Threads);
    for (int pass = 0; pass < 2; ++pass) {
        k_r2_partial<<<nb, kR2Threads, 0, s>>>(truth, approx, origin, numel, pass, ws);
        k_r2_final<<<1, 32, 0, s>>>(pass, nb, ws);
    }
    cudaError_t e = cudaMemcpyAsync(r2, ws + 1, sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return csd::cuda_status(e, "r_squared");
    c->launches += 4;
    if (std::isnan(*r2)) return set_error(CSD_ERR_NUMERIC, "r_squared undefined: true delta has zero variance");
    return CSD_OK;
}

csd_status csd_index_set_to_masks(csd_ctx* ctx, const int32_t* idx, const int32_t* counts,
                                  int64_t rows, int64_t k_max, int64_t n_bits, uint8_t* masks,
                                  void* stream) {
    if (!ctx) return set_error(CSD_ERR_VALUE, "null context");
    if (rows < 0 || k_max < 0 || n_bits < 0)
        return set_error(CSD_ERR_SHAPE, "index_set_to_masks: negative extent");
    if (k_max > n_bits)
        return set_error(CSD_ERR_VALUE, "mask length %lld smaller than index k_max %lld",
                         (long long)n_bits, (long long)k_max);
    if (rows == 0) return CSD_OK;
    auto* c = reinterpret_cast<csd::Ctx*>(ctx);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t row_bytes = (n_bits + 7) / 8;
    const size_t smem = (size_t)((n_bits + 31) / 32) * 4 + 4;
    if (smem > 200 * 1024)
        return set_error(CSD_ERR_UNSUPPORTED, "mask length %lld too long", (long long)n_bits);
    static size_t attr = 48 * 1024;  // opt in once per larger size (keeps graph capture clean)
    if (smem > attr) {
        CSD_CU_(cudaFuncSetAttribute(csd::dev::k_index_masks,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = smem;
    }
    csd::dev::k_index_masks<<<(unsigned)rows, 256, smem, s>>>(idx, counts, k_max, n_bits,
                                                              row_bytes, masks, c->flags);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return csd::cuda_status(e, "index_set_to_masks");
    c->launches += 1;
    return csd::check_flags(c, s);  // the reference validates first (IndexError / ValueError)
}

}  // extern "C"
