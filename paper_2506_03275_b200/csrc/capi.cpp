// capi.cpp — the C ABI (include/csd_b200.h): validation with the reference's
// error semantics, workspace management, mode dispatch to the CUDA kernels.
//
// No entry point ever computes on the host: CHECK mode dispatches to the
// bit-exact CUDA kernels (check_kernels.cu), PROD mode to the tcgen05 / bf16
// kernels (attn_tc.cu, prod_kernels.cu) and cuBLAS for plain dense GEMMs.
#include "capi_internal.h"

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace csd::dev;

namespace {
thread_local std::string g_last_error;
}

namespace csd {

csd_status set_error(csd_status s, const char* fmt, ...) {
    if (s == CSD_OK) return s;
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

csd_status cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return CSD_OK;
    if (e == cudaErrorNotSupported)
        return set_error(CSD_ERR_UNSUPPORTED, "%s: shape outside the production kernel envelope",
                         where);
    return set_error(CSD_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

void* Ctx::ws(int slot, size_t bytes, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(mu);
    if (slot >= (int)bufs.size()) bufs.resize(slot + 1, {nullptr, 0});
    auto& b = bufs[slot];
    if (b.second < bytes) {
        // Growing during stream capture would put an allocation inside the captured region
        // (and the new pointer would only be valid for this graph): refuse.
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (s != nullptr && cudaStreamIsCapturing(s, &cs) == cudaSuccess &&
            cs != cudaStreamCaptureStatusNone) {
            set_error(CSD_ERR_CUDA,
                      "workspace slot %d must grow to %zu bytes during stream capture: run the "
                      "step once eagerly before capturing it", slot, bytes);
            return nullptr;
        }
        // The old buffer is NOT freed: CUDA graphs captured earlier may still read and write
        // it.  Retired buffers live until csd_ctx_destroy.
        if (b.first) retired.push_back(b.first);
        b.first = nullptr;
        b.second = 0;
        if (cudaMalloc(&b.first, bytes < 256 ? 256 : bytes) != cudaSuccess) return nullptr;
        b.second = bytes;
    }
    return b.first;
}

cublasHandle_t Ctx::blas() {
    if (!cublas) {
        cublasCreate(&cublas);
        cublasSetMathMode(cublas, CUBLAS_DEFAULT_MATH);
    }
    return cublas;
}

// Row-major bf16 GEMMs through cuBLAS (column-major) — plain library GEMMs only.
// C[M,N] = A[M,K] @ B   with B given as [N,K] (b_nk = true) or [K,N].
csd_status gemm_bf16(Ctx* ctx, const void* a, const void* b, bool b_nk, void* c, bool c_f32,
                     int64_t m, int64_t n, int64_t k, float beta, cudaStream_t s) {
    cublasHandle_t h = ctx->blas();
    cublasSetStream(h, s);
    const float alpha = 1.0f;
    // column-major: C^T[N,M] = op(B)[N,K] * A^T[K,M]
    cublasStatus_t st = cublasGemmEx(
        h, b_nk ? CUBLAS_OP_T : CUBLAS_OP_N, CUBLAS_OP_N, (int)n, (int)m, (int)k, &alpha, b,
        CUDA_R_16BF, b_nk ? (int)k : (int)n, a, CUDA_R_16BF, (int)k, &beta, c,
        c_f32 ? CUDA_R_32F : CUDA_R_16BF, (int)n, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    if (st != CUBLAS_STATUS_SUCCESS) return set_error(CSD_ERR_CUDA, "cublasGemmEx failed (%d)", (int)st);
    ctx->library_launches += 1;
    return CSD_OK;
}

// Per-chunk GEMM over the chunk-major activation cache [B*C, F, chunk] (mlp_tc.cu layout):
// out[z*chunk + r, :] = sum_f cm[z, f, r] * W2[f, :] for every chunk z, as one strided-
// batched call (A^T of each chunk is the contiguous [F, chunk] slab; W2 shared).
csd_status gemm_bf16_chunks(Ctx* ctx, const void* cm, const void* w2, void* out, bool c_f32,
                            int64_t chunks, int64_t chunk, int64_t d, int64_t f, cudaStream_t s) {
    cublasHandle_t h = ctx->blas();
    cublasSetStream(h, s);
    const float alpha = 1.0f, beta = 0.0f;
    // column-major per chunk: C^T[D, chunk] = W2^T[D, F] * (act_z)^T[F, chunk], act_z being the
    // column-major [chunk, F] view of the [F, chunk] slab (ld = chunk, op T)
    cublasStatus_t st = cublasGemmStridedBatchedEx(
        h, CUBLAS_OP_N, CUBLAS_OP_T, (int)d, (int)chunk, (int)f, &alpha, w2, CUDA_R_16BF, (int)d,
        0, cm, CUDA_R_16BF, (int)chunk, f * chunk, &beta, out, c_f32 ? CUDA_R_32F : CUDA_R_16BF,
        (int)d, chunk * d, (int)chunks, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    if (st != CUBLAS_STATUS_SUCCESS)
        return set_error(CSD_ERR_CUDA, "cublasGemmStridedBatchedEx failed (%d)", (int)st);
    ctx->library_launches += 1;
    return CSD_OK;
}

csd_status check_flags(Ctx* ctx, cudaStream_t s) {
    uint32_t f = 0;
    cudaError_t e = cudaMemcpyAsync(&f, ctx->flags, sizeof(f), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e, "csd_ctx_sync");
    if (f) cudaMemsetAsync(ctx->flags, 0, sizeof(uint32_t), s);
    if (f & kFlagIndexRange) return set_error(CSD_ERR_INDEX, "sparse index out of range");
    if (f & kFlagIndexDup) return set_error(CSD_ERR_INDEX, "duplicate sparse index within one chunk");
    if (f & kFlagCountRange) return set_error(CSD_ERR_VALUE, "sparse index count outside [0, k_max]");
    if (f & kFlagNonFinite) return set_error(CSD_ERR_NUMERIC, "softmax_rows: non-finite logit");
    return CSD_OK;
}

}  // namespace csd

using csd::Ctx;
using csd::set_error;
using csd::cuda_status;

#define CSD_TRY(expr)                          \
    do {                                       \
        csd_status _s = (expr);                \
        if (_s != CSD_OK) return _s;           \
    } while (0)
#define CSD_CU(expr, where)                                  \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) return cuda_status(_e, where); \
    } while (0)

static inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" {

int csd_abi_version(void) { return CSD_ABI_VERSION; }
const char* csd_last_error(void) { return g_last_error.c_str(); }
const char* csd_status_name(csd_status s) {
    switch (s) {
        case CSD_OK: return "OK";
        case CSD_ERR_SHAPE: return "ShapeError";
        case CSD_ERR_INDEX: return "IndexError";
        case CSD_ERR_NUMERIC: return "NumericError";
        case CSD_ERR_STATE: return "StateError";
        case CSD_ERR_VALUE: return "ValueError";
        case CSD_ERR_CONFIG: return "ConfigError";
        case CSD_ERR_CUDA: return "CudaError";
        case CSD_ERR_UNSUPPORTED: return "Unsupported";
    }
    return "Unknown";
}

csd_status csd_ctx_create(int device, csd_ctx** out) {
    if (!out) return set_error(CSD_ERR_VALUE, "csd_ctx_create: null out");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) return set_error(CSD_ERR_CUDA, "no CUDA device visible");
    if (device < 0 || device >= n) return set_error(CSD_ERR_VALUE, "device %d out of range", device);
    CSD_CU(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    CSD_CU(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10)
        return set_error(CSD_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a",
                         device, prop.major, prop.minor);
    auto* c = new Ctx;
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    if (cudaMalloc(&c->flags, sizeof(uint32_t)) != cudaSuccess) {
        delete c;
        return set_error(CSD_ERR_CUDA, "cudaMalloc(flags) failed");
    }
    cudaMemset(c->flags, 0, sizeof(uint32_t));
    *out = reinterpret_cast<csd_ctx*>(c);
    return CSD_OK;
}

csd_status csd_ctx_destroy(csd_ctx* ctx) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    if (!c) return CSD_OK;
    cudaDeviceSynchronize();
    for (auto& b : c->bufs)
        if (b.first) cudaFree(b.first);
    for (void* p : c->retired) cudaFree(p);
    if (c->flags) cudaFree(c->flags);
    if (c->cublas) cublasDestroy(c->cublas);
    delete c;
    return CSD_OK;
}

csd_status csd_ctx_sync(csd_ctx* ctx, void* stream) {
    return csd::check_flags(reinterpret_cast<Ctx*>(ctx), S(stream));
}

int64_t csd_ctx_launch_count(const csd_ctx* ctx) {
    return reinterpret_cast<const Ctx*>(ctx)->launches;
}

// ---------------------------------------------------------------- voxel
csd_status csd_voxel_permutation(int64_t t, int64_t h, int64_t w, int64_t vt, int64_t vh,
                                 int64_t vw, int64_t* perm) {
    // voxel.cpp:7-16 validation, :18-42 enumeration (host: it is a plan, not data)
    if (t < 1 || h < 1 || w < 1 || vt < 1 || vh < 1 || vw < 1)
        return set_error(CSD_ERR_CONFIG, "voxel layout dimensions must be >= 1");
    if (t % vt || h % vh || w % vw)
        return set_error(CSD_ERR_CONFIG, "voxel (%lld,%lld,%lld) does not tile grid (%lld,%lld,%lld)",
                         (long long)vt, (long long)vh, (long long)vw, (long long)t, (long long)h,
                         (long long)w);
    int64_t pos = 0;
    for (int64_t tc = 0; tc < t / vt; ++tc)
        for (int64_t hc = 0; hc < h / vh; ++hc)
            for (int64_t wc = 0; wc < w / vw; ++wc)
                for (int64_t it = 0; it < vt; ++it)
                    for (int64_t ih = 0; ih < vh; ++ih)
                        for (int64_t iw = 0; iw < vw; ++iw)
                            perm[pos++] = ((tc * vt + it) * h + hc * vh + ih) * w + wc * vw + iw;
    return CSD_OK;
}

csd_status csd_voxel_reorder(csd_ctx* ctx, const void* src, void* dst, int64_t batch, int64_t t,
                             int64_t h, int64_t w, int64_t vt, int64_t vh, int64_t vw,
                             int64_t row_bytes, int inverse, void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    if (t < 1 || h < 1 || w < 1 || vt < 1 || vh < 1 || vw < 1)
        return set_error(CSD_ERR_CONFIG, "voxel layout dimensions must be >= 1");
    if (t % vt || h % vh || w % vw)
        return set_error(CSD_ERR_CONFIG, "voxel (%lld,%lld,%lld) does not tile grid (%lld,%lld,%lld)",
                         (long long)vt, (long long)vh, (long long)vw, (long long)t, (long long)h,
                         (long long)w);
    if (batch < 1 || row_bytes < 1) return set_error(CSD_ERR_SHAPE, "voxel reorder: empty tensor");
    if (src == dst) return set_error(CSD_ERR_VALUE, "voxel reorder cannot run in place");
    CSD_CU(voxel_reorder(src, dst, batch, t, h, w, vt, vh, vw, row_bytes, inverse, S(stream)),
           "voxel_reorder");
    c->launches += 1;
    return CSD_OK;
}

// ---------------------------------------------------------------- top-k
csd_status csd_select_top_k(csd_ctx* ctx, const float* scores, int64_t rows, int64_t m, int64_t k,
                            int32_t* idx, int32_t* counts, void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    if (k < 1 || k > m)
        return set_error(CSD_ERR_VALUE, "select_top_k: k=%lld outside [1, %lld]", (long long)k,
                         (long long)m);
    if (rows < 1) return set_error(CSD_ERR_SHAPE, "select_top_k: no rows");
    if (k <= topk_max_k()) {
        CSD_CU(topk_rows(scores, rows, m, k, idx, counts, S(stream), c->sorted_topk), "topk_rows");
        c->launches += 1;
    } else {
        void* ws = c->ws(csd::kWsTopk, sizeof(uint64_t) * rows * k, S(stream));
        if (!ws) return set_error(CSD_ERR_CUDA, "workspace allocation failed");
        CSD_CU(topk_rows_global(scores, rows, m, k, idx, counts, (uint64_t*)ws, S(stream)),
               "topk_rows_global");
        c->launches += 2;
    }
    return CSD_OK;
}

csd_status csd_validate_index_set(csd_ctx* ctx, const int32_t* idx, const int32_t* counts,
                                  int64_t rows, int64_t k_max, int64_t domain, void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    if (k_max < 0 || k_max > domain)
        return set_error(CSD_ERR_VALUE, "sparse index set k_max %lld outside [0, domain=%lld]",
                         (long long)k_max, (long long)domain);
    CSD_CU(validate_index_set(idx, counts, rows, k_max, domain, c->flags, S(stream)), "validate");
    c->launches += 1;
    return CSD_OK;
}

}  // extern "C"
