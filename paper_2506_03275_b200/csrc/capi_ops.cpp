// capi_ops.cpp — attention / MLP / dense-op entry points of the C ABI.
//
// CHECK mode mirrors the reference's exception semantics exactly: index sets
// are validated (on device) BEFORE any output is written and the call is
// synchronous, returning the status the reference would have thrown.  PROD
// mode is fully asynchronous; index validation (if enabled) runs as one small
// kernel whose verdict surfaces at csd_ctx_sync().
#include <cmath>
#include <cstring>

#include "capi_internal.h"

using namespace csd::dev;
using csd::Ctx;
using csd::cuda_status;
using csd::set_error;

#define CSD_TRY(expr)                \
    do {                             \
        csd_status _s = (expr);      \
        if (_s != CSD_OK) return _s; \
    } while (0)
#define CSD_CU(expr, where)                                   \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) return cuda_status(_e, where); \
    } while (0)

namespace {

inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

csd_status need_ws(void* p) {
    return p ? CSD_OK : set_error(CSD_ERR_CUDA, "workspace allocation failed");
}

csd_status check_attn_shape(int64_t b, int64_t h, int64_t n, int64_t e, int layout) {
    if (b < 1 || h < 1 || n < 1 || e < 1)
        return set_error(CSD_ERR_SHAPE, "attention expects [B x H x N x E] with all dims >= 1");
    if (layout != CSD_LAYOUT_BHNE && layout != CSD_LAYOUT_BNHE)
        return set_error(CSD_ERR_VALUE, "unknown attention layout %d", layout);
    return CSD_OK;
}

csd_status check_chunk(int64_t n, int64_t chunk, const char* who) {
    if (chunk < 1 || n % chunk != 0)
        return set_error(CSD_ERR_SHAPE, "%s: sequence length %lld not divisible by chunk %lld", who,
                         (long long)n, (long long)chunk);
    return CSD_OK;
}

csd_status sync_validate(Ctx* c, const int32_t* idx, const int32_t* counts, int64_t rows,
                         int64_t k_max, int64_t domain, cudaStream_t s) {
    if (k_max < 0 || k_max > domain)
        return set_error(CSD_ERR_VALUE, "sparse index set k_max %lld outside [0, domain=%lld]",
                         (long long)k_max, (long long)domain);
    CSD_CU(validate_index_set(idx, counts, rows, k_max, domain, c->flags, s), "validate");
    c->launches += 1;
    return csd::check_flags(c, s);
}

csd_status prod_attn(Ctx* c, const AttnTcArgs& a, cudaStream_t s) {
    if (!attn_tc_supported(a.e, a.chunk))
        return set_error(CSD_ERR_UNSUPPORTED,
                         "production attention supports head_dim 64/128 and chunk <= 256 "
                         "(got E=%lld, chunk=%lld)",
                         (long long)a.e, (long long)a.chunk);
    CSD_CU(attn_tc(a, s), "attn_tc");
    c->launches += 1;
    return CSD_OK;
}

}  // namespace

namespace csd {
// Dense MLP, PROD (mlp.cpp:49-81): cuBLAS GEMM1 -> bf16 pre; fused bias+GELU writing the
// chunk-major cache (+ row-major activations when chunk > 256); cuBLAS GEMM2 (per chunk over
// the cache) -> fp32 M_cache; fused
// +b2 (and, for the block runner, x_out = x_mid + M_cache).
csd_status prod_dense_mlp(Ctx* c, const void* x, const void* w1, const float* b1, const void* w2,
                          const float* b2, int64_t batch, int64_t n, int64_t d, int64_t f,
                          int64_t chunk, float* out, void* act_cm, const void* x_mid, void* x_out,
                          cudaStream_t s) {
    const int64_t rows = batch * n;
    if (gemm_tc_enabled() && gemm_tc_mlp_supported(d, f, chunk)) {
        // hand-written tcgen05 GEMMs (gemm_tc.cu): GEMM1 writes gelu(x W1^T + b1) straight
        // into the chunk-major cache, GEMM2 reads it and writes M_cache (+b2) and x_out
        if (!act_cm) {
            act_cm = c->ws(kWsScores, 2 * rows * f, s);
            CSD_TRY(need_ws(act_cm));
        }
        CSD_CU(gemm_tc_mlp_up(x, w1, b1, batch * (n / chunk), chunk, d, f, act_cm, s), "gemm_tc_mlp_up");
        CSD_CU(gemm_tc_mlp_down(act_cm, w2, b2, batch * (n / chunk), chunk, d, f, out, x_mid, x_out, s),
               "gemm_tc_mlp_down");
        c->launches += 2;
        return CSD_OK;
    }
    // chunk <= 256: GELU writes only the chunk-major cache and GEMM2 runs per chunk over it
    // (saves the [rows, F] row-major activation write); otherwise the row-major path
    const bool from_cm = chunk <= 256;
    void* pre = c->ws(kWsPre, 2 * rows * f, s);
    CSD_TRY(need_ws(pre));
    void* act = nullptr;
    if (!from_cm) {
        act = c->ws(kWsAct, 2 * rows * f, s);
        CSD_TRY(need_ws(act));
    }
    if (!act_cm) {
        act_cm = c->ws(kWsScores, 2 * rows * f, s);
        CSD_TRY(need_ws(act_cm));
    }
    CSD_TRY(gemm_bf16(c, x, w1, true, pre, false, rows, f, d, 0.0f, s));
    CSD_CU(prod_bias_gelu_cm(pre, b1, batch, n, f, chunk, act, act_cm, s), "bias_gelu_cm");
    if (from_cm)
        CSD_TRY(gemm_bf16_chunks(c, act_cm, w2, out, true, batch * (n / chunk), chunk, d, f, s));
    else
        CSD_TRY(gemm_bf16(c, act, w2, false, out, true, rows, d, f, 0.0f, s));
    CSD_CU(prod_bias_add_rows(out, b2, rows, d, x_mid, x_out, s), "bias_add");
    c->launches += 2;
    return CSD_OK;
}
}  // namespace csd

extern "C" {

csd_status csd_ctx_set_validation(csd_ctx* ctx, int enabled) {
    reinterpret_cast<Ctx*>(ctx)->validate_prod = enabled != 0;
    return CSD_OK;
}

csd_status csd_ctx_set_lpt(csd_ctx* ctx, int enabled) {
    if (!ctx) return set_error(CSD_ERR_VALUE, "null context");
    reinterpret_cast<Ctx*>(ctx)->lpt = enabled != 0;
    return CSD_OK;
}

csd_status csd_ctx_set_sorted_topk(csd_ctx* ctx, int sorted) {
    if (!ctx) return set_error(CSD_ERR_VALUE, "null context");
    reinterpret_cast<Ctx*>(ctx)->sorted_topk = sorted != 0;
    return CSD_OK;
}

// ---------------------------------------------------------------- attention
csd_status csd_dense_attention(csd_ctx* ctx, csd_mode mode, csd_layout layout, const void* q,
                               const void* k, const void* v, int64_t batch, int64_t heads,
                               int64_t n, int64_t e, void* out, void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    CSD_TRY(check_attn_shape(batch, heads, n, e, layout));
    const cudaStream_t s = S(stream);
    if (mode == CSD_MODE_PROD) {
        AttnTcArgs a{};
        a.q = q; a.k = k; a.v = v; a.out = out; a.layout = layout;
        a.batch = batch; a.heads = heads; a.n = n; a.e = e;
        // query rows per work item: the widest tiling that divides N — 256 rows keep both
        // M-tiles of a CTA live (the two tiles' softmax and MMAs ping-pong); measured on the
        // FLUX shape: 256 -> 0.32 ms, 192 -> 0.41 ms, 128 -> 0.50 ms
        a.chunk = 0;
        for (int64_t cc : {256, 192, 128})
            if (n % cc == 0) { a.chunk = cc; break; }
        if (a.chunk == 0) {  // any divisor <= 256 works for a dense pass
            for (int64_t cc = 256; cc >= 1; --cc)
                if (n % cc == 0) { a.chunk = cc; break; }
        }
        return prod_attn(c, a, s);
    }
    const int64_t bh = batch * heads;
    float* L = (float*)c->ws(csd::kWsLogits, sizeof(float) * bh * n * n, s);
    float* P = (float*)c->ws(csd::kWsProbs, sizeof(float) * bh * n * n, s);
    CSD_TRY(need_ws(L));
    CSD_TRY(need_ws(P));
    CSD_CU(check_attention_logits((const float*)q, (const float*)k, layout, batch, heads, n, e, n,
                                  nullptr, nullptr, 0, L, s), "logits");
    CSD_CU(cudaMemcpyAsync(P, L, sizeof(float) * bh * n * n, cudaMemcpyDeviceToDevice, s), "copy");
    CSD_CU(check_softmax(P, bh * n, n, n, nullptr, n, nullptr, nullptr, c->flags, s), "softmax");
    CSD_CU(check_attention_pv(P, (const float*)v, layout, batch, heads, n, e, n, nullptr, nullptr,
                              0, nullptr, 1.0f, (float*)out, s), "pv");
    c->launches += 2 + bh * 2;
    return csd::check_flags(c, s);
}

csd_status csd_column_sum_attention(csd_ctx* ctx, csd_mode mode, csd_layout layout,
                                    const void* q, const void* k, const void* v,
                                    const float* prev_m, const float* prev_l, int64_t batch,
                                    int64_t heads, int64_t n, int64_t e, int64_t chunk, void* out,
                                    float* row_max, float* exp_sum, float* column_sums,
                                    void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    CSD_TRY(check_attn_shape(batch, heads, n, e, layout));
    CSD_TRY(check_chunk(n, chunk, "column_sum_attention"));
    if ((prev_m == nullptr) != (prev_l == nullptr))
        return set_error(CSD_ERR_SHAPE, "column_sum_attention: previous stats need both m and l");
    const cudaStream_t s = S(stream);
    if (mode == CSD_MODE_PROD) {
        AttnTcArgs a{};
        a.q = q; a.k = k; a.v = v; a.out = out; a.layout = layout;
        a.batch = batch; a.heads = heads; a.n = n; a.e = e; a.chunk = chunk;
        a.row_max = row_max; a.exp_sum = exp_sum;
        // 256-row work items keep both M-tiles live (the dense kernel's best tiling, FLUX
        // 0.32 vs 0.41 ms at 192 rows); the column sums stay per `chunk` rows.  chunk >= 128
        // keeps every item within two chunks (the kernel's order-independent atomic merge)
        if (chunk >= 128 && chunk < 256 && chunk % 32 == 0 && n % 256 == 0) {
            a.chunk = 256;
            a.cs_chunk = chunk;  // the kernels that merge partial column sums zero the buffer
        }
        if (prev_m == nullptr) {
            // first dense step: exact probabilities need the final stats first
            CSD_TRY(prod_attn(c, a, s));
            a.prev_m = row_max; a.prev_l = exp_sum;
            a.row_max = nullptr; a.exp_sum = nullptr;
        } else {
            a.prev_m = prev_m; a.prev_l = prev_l;
        }
        a.colsum = column_sums;
        return prod_attn(c, a, s);
    }
    const int64_t bh = batch * heads;
    float* L = (float*)c->ws(csd::kWsLogits, sizeof(float) * bh * n * n, s);
    float* P = (float*)c->ws(csd::kWsProbs, sizeof(float) * bh * n * n, s);
    CSD_TRY(need_ws(L));
    CSD_TRY(need_ws(P));
    CSD_CU(check_attention_logits((const float*)q, (const float*)k, layout, batch, heads, n, e, n,
                                  nullptr, nullptr, 0, L, s), "logits");
    CSD_CU(cudaMemcpyAsync(P, L, sizeof(float) * bh * n * n, cudaMemcpyDeviceToDevice, s), "copy");
    CSD_CU(check_softmax(P, bh * n, n, n, nullptr, n, row_max, exp_sum, c->flags, s), "softmax");
    CSD_CU(check_attention_pv(P, (const float*)v, layout, batch, heads, n, e, n, nullptr, nullptr,
                              0, nullptr, 1.0f, (float*)out, s), "pv");
    CSD_CU(check_colsum(L, prev_m ? prev_m : row_max, prev_l ? prev_l : exp_sum, bh, n, chunk,
                        column_sums, s), "colsum");
    c->launches += 3 + bh * 2;
    return csd::check_flags(c, s);
}

csd_status csd_sparse_delta_attention(csd_ctx* ctx, csd_mode mode, csd_layout layout,
                                      const void* q, const void* k, const void* v,
                                      const int32_t* idx, const int32_t* counts, int64_t k_max,
                                      int64_t chunk, const void* base, float scale,
                                      int64_t batch, int64_t heads, int64_t n, int64_t e,
                                      void* out, void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    CSD_TRY(check_attn_shape(batch, heads, n, e, layout));
    CSD_TRY(check_chunk(n, chunk, "sparse_delta_attention"));
    const cudaStream_t s = S(stream);
    const int64_t nc = n / chunk;
    const int64_t rows = batch * heads * nc;
    if (mode == CSD_MODE_PROD) {
        if (c->validate_prod) {
            if (k_max < 0 || k_max > n)
                return set_error(CSD_ERR_VALUE, "sparse index set k_max %lld outside [0, domain=%lld]",
                                 (long long)k_max, (long long)n);
            CSD_CU(validate_index_set(idx, counts, rows, k_max, n, c->flags, s), "validate");
            c->launches += 1;
        }
        AttnTcArgs a{};
        a.q = q; a.k = k; a.v = v; a.idx = idx; a.counts = counts; a.k_max = k_max;
        a.base = base; a.scale = scale; a.out = out; a.layout = layout;
        a.batch = batch; a.heads = heads; a.n = n; a.e = e; a.chunk = chunk;
        if (c->lpt && attn_pp_supported(a) && k_max > 128) {
            // ragged counts: longest items first over the persistent CTAs
            auto* order = static_cast<int32_t*>(c->ws(csd::kWsOrder, sizeof(int32_t) * (rows + 1), s));
            CSD_TRY(need_ws(order));
            CSD_CU(lpt_order(counts, rows, 128, order, s), "lpt_order");
            c->launches += 1;
            a.order = order;
        }
        return prod_attn(c, a, s);
    }
    CSD_TRY(sync_validate(c, idx, counts, rows, k_max, n, s));
    const size_t bytes = sizeof(float) * batch * heads * n * e;
    if (out != base) CSD_CU(cudaMemcpyAsync(out, base, bytes, cudaMemcpyDeviceToDevice, s), "copy");
    if (k_max == 0) return CSD_OK;
    float* L = (float*)c->ws(csd::kWsLogits, sizeof(float) * batch * heads * n * k_max, s);
    CSD_TRY(need_ws(L));
    CSD_CU(check_attention_logits((const float*)q, (const float*)k, layout, batch, heads, n, e,
                                  chunk, idx, counts, k_max, L, s), "logits");
    CSD_CU(check_softmax(L, batch * heads * n, chunk, k_max, counts, k_max, nullptr, nullptr,
                         c->flags, s), "softmax");
    CSD_CU(check_attention_pv(L, (const float*)v, layout, batch, heads, n, e, chunk, idx, counts,
                              k_max, (const float*)base == (const float*)out ? (const float*)out
                                                                             : (const float*)base,
                              scale, (float*)out, s), "pv");
    c->launches += 2 + batch * heads;
    return csd::check_flags(c, s);
}

// ---------------------------------------------------------------- MLP
static csd_status check_mlp_shape(int64_t b, int64_t n, int64_t d, int64_t f) {
    if (b < 1 || n < 1 || d < 1 || f < 1)
        return set_error(CSD_ERR_SHAPE, "mlp expects [B x N x D] input and [F x D] weights");
    return CSD_OK;
}

csd_status csd_dense_mlp(csd_ctx* ctx, csd_mode mode, const void* x, const void* w1,
                         const float* b1, const void* w2, const float* b2, int64_t batch,
                         int64_t n, int64_t d, int64_t f, int64_t chunk, float* out,
                         void* act_out, void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    CSD_TRY(check_mlp_shape(batch, n, d, f));
    const cudaStream_t s = S(stream);
    const int64_t rows = batch * n;
    if (mode == CSD_MODE_PROD) {
        CSD_TRY(check_chunk(n, chunk, "dense_mlp"));
        return csd::prod_dense_mlp(c, x, w1, b1, w2, b2, batch, n, d, f, chunk, out, act_out,
                                   nullptr, nullptr, s);
    }
    float* act = act_out ? (float*)act_out : (float*)c->ws(csd::kWsAct, sizeof(float) * rows * f, s);
    CSD_TRY(need_ws(act));
    CSD_CU(check_dense_mlp((const float*)x, (const float*)w1, b1, (const float*)w2, b2, batch, n, d,
                           f, act, out, s), "dense_mlp");
    c->launches += 2;
    return csd::check_flags(c, s);
}

csd_status csd_mlp_tile_means(csd_ctx* ctx, csd_mode mode, const void* x, const void* w1,
                              int64_t batch, int64_t n, int64_t d, int64_t f, int64_t chunk,
                              float* out, void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    CSD_TRY(check_mlp_shape(batch, n, d, f));
    CSD_TRY(check_chunk(n, chunk, "mlp_tile_means"));
    const cudaStream_t s = S(stream);
    if (mode == CSD_MODE_PROD) {
        if (!means_tc_supported(d, f))
            return set_error(CSD_ERR_UNSUPPORTED, "production tile means need D %% 64 == 0 and F %% 128 == 0");
        void* ws = c->ws(csd::kWsMeans, prod_means_ws_bytes(batch, n, d, f, chunk), s);
        CSD_TRY(need_ws(ws));
        CSD_CU(prod_tile_means_tc(x, w1, batch, n, d, f, chunk, nullptr, out, ws, s), "tile_means");
        c->launches += 3;
        return CSD_OK;
    }
    float* means = (float*)c->ws(csd::kWsMeans, sizeof(float) * batch * (n / chunk) * d, s);
    CSD_TRY(need_ws(means));
    CSD_CU(check_tile_means((const float*)x, (const float*)w1, batch, n, d, f, chunk, means, out, s),
           "tile_means");
    c->launches += 2;
    return CSD_OK;
}

csd_status csd_mlp_change_indices(csd_ctx* ctx, csd_mode mode, const void* x, const void* w1,
                                  const float* tile_means, int64_t batch, int64_t n, int64_t d,
                                  int64_t f, int64_t k, int64_t chunk, int32_t* idx,
                                  int32_t* counts, void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    CSD_TRY(check_mlp_shape(batch, n, d, f));
    CSD_TRY(check_chunk(n, chunk, "mlp_change_indices"));
    if (k < 1 || k > f)
        return set_error(CSD_ERR_VALUE, "mlp_change_indices: k=%lld outside [1, %lld]", (long long)k,
                         (long long)f);
    const cudaStream_t s = S(stream);
    const int64_t rows = batch * (n / chunk);
    float* scores = (float*)c->ws(csd::kWsScores, sizeof(float) * rows * f * 2, s);
    CSD_TRY(need_ws(scores));
    if (mode == CSD_MODE_PROD) {
        if (!means_tc_supported(d, f))
            return set_error(CSD_ERR_UNSUPPORTED, "production tile means need D %% 64 == 0 and F %% 128 == 0");
        void* ws = c->ws(csd::kWsMeans, prod_means_ws_bytes(batch, n, d, f, chunk), s);
        CSD_TRY(need_ws(ws));
        if (!c->sorted_topk && topk_cluster_eligible(rows, f) && k <= f) {
            // unsorted selection: |T - T_m| reduced inside the cluster top-k's load
            MeansPartials mp{};
            CSD_CU(prod_tile_means_tc(x, w1, batch, n, d, f, chunk, tile_means, scores, ws, s, &mp),
                   "tile_means");
            CSD_CU(topk_rows_fused_absdiff(mp.partial, mp.ks, tile_means, rows, f, k, idx, counts, s),
                   "topk_fused");
            c->launches += 3;
            return CSD_OK;
        }
        // |tile_means(x) - T_m| fused into the split-K reduction (mlp.cpp:116)
        CSD_CU(prod_tile_means_tc(x, w1, batch, n, d, f, chunk, tile_means, scores, ws, s),
               "tile_means");
        c->launches += 3;
    } else {
        float* fresh = scores + rows * f;
        CSD_TRY(csd_mlp_tile_means(ctx, mode, x, w1, batch, n, d, f, chunk, fresh, stream));
        CSD_CU(check_absdiff(fresh, tile_means, rows * f, scores, s), "absdiff");
        c->launches += 1;
    }
    return csd_select_top_k(ctx, scores, rows, f, k, idx, counts, stream);
}

csd_status csd_sparse_delta_mlp(csd_ctx* ctx, csd_mode mode, const void* x, const void* w1,
                                const float* b1, const void* w2, const int32_t* idx,
                                const int32_t* counts, int64_t k_max, int64_t chunk,
                                int64_t batch, int64_t n, int64_t d, int64_t f, void* act_cache,
                                float* out_cache, void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    CSD_TRY(check_mlp_shape(batch, n, d, f));
    CSD_TRY(check_chunk(n, chunk, "sparse_delta_mlp"));
    const cudaStream_t s = S(stream);
    const int64_t rows = batch * (n / chunk);
    if (mode == CSD_MODE_PROD) {
        if (c->validate_prod) {
            if (k_max < 0 || k_max > f)
                return set_error(CSD_ERR_VALUE, "sparse index set k_max %lld outside [0, domain=%lld]",
                                 (long long)k_max, (long long)f);
            CSD_CU(validate_index_set(idx, counts, rows, k_max, f, c->flags, s), "validate");
            c->launches += 1;
        }
        if (!mlp_tc_supported(d, chunk))
            return set_error(CSD_ERR_UNSUPPORTED,
                             "production sparse-delta MLP needs model_dim %% 128 == 0 and chunk <= 256 "
                             "(got D=%lld, chunk=%lld)", (long long)d, (long long)chunk);
        const int64_t k_pad = csd::dev::prod_smlp_delta_cols(k_max, rows, chunk);
        void* dws = c->ws(csd::kWsDelta, 2 * rows * chunk * (k_pad ? k_pad : 128), s);
        CSD_TRY(need_ws(dws));
        CSD_CU(prod_sparse_delta_mlp_tc(x, w1, b1, w2, idx, counts, k_max, chunk, batch, n, d, f,
                                        act_cache, out_cache, dws, s), "sparse_delta_mlp");
        c->launches += 2;
        return CSD_OK;
    }
    CSD_TRY(sync_validate(c, idx, counts, rows, k_max, f, s));
    if (k_max == 0) return CSD_OK;
    float* ws = (float*)c->ws(csd::kWsDelta, sizeof(float) * rows * chunk * k_max, s);
    CSD_TRY(need_ws(ws));
    CSD_CU(check_sparse_delta_mlp((const float*)x, (const float*)w1, b1, (const float*)w2, idx,
                                  counts, k_max, chunk, batch, n, d, f, (float*)act_cache,
                                  out_cache, ws, s), "sparse_delta_mlp");
    c->launches += 3;
    return csd::check_flags(c, s);
}

csd_status csd_mlp_act_cache_to_ref(csd_ctx* ctx, csd_mode mode, const void* act_cache,
                                    int64_t batch, int64_t n, int64_t f, int64_t chunk,
                                    float* out, void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    CSD_TRY(check_chunk(n, chunk, "act_cache_to_ref"));
    const cudaStream_t s = S(stream);
    if (mode == CSD_MODE_PROD) {
        CSD_CU(prod_act_cm_to_ref(act_cache, batch, n, f, chunk, out, s), "cm_to_ref");
        c->launches += 1;
        return CSD_OK;
    }
    if (act_cache != out)
        CSD_CU(cudaMemcpyAsync(out, act_cache, sizeof(float) * batch * n * f,
                               cudaMemcpyDeviceToDevice, s), "copy");
    return CSD_OK;
}

// ---------------------------------------------------------------- dense ops
csd_status csd_project(csd_ctx* ctx, csd_mode mode, const void* x, const void* w, int64_t batch,
                       int64_t n, int64_t d, int64_t dout, void* out, void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    if (batch < 1 || n < 1 || d < 1 || dout < 1)
        return set_error(CSD_ERR_SHAPE, "project expects [B x N x D] input");
    const cudaStream_t s = S(stream);
    if (mode == CSD_MODE_PROD) {
        if (gemm_tc_enabled() && gemm_tc_proj_supported(batch * n, d, dout)) {
            const void* ws[3] = {w, w, w};
            void* os[3] = {out, out, out};
            CSD_CU(gemm_tc_proj(x, ws, os, 1, batch * n, d, dout, nullptr, s), "gemm_tc_proj");
            c->launches += 1;
            return CSD_OK;
        }
        return csd::gemm_bf16(c, x, w, false, out, false, batch * n, dout, d, 0.0f, s);
    }
    CSD_CU(check_project((const float*)x, (const float*)w, batch, n, d, dout, (float*)out, s),
           "project");
    c->launches += 1;
    return CSD_OK;
}

csd_status csd_add(csd_ctx* ctx, csd_mode mode, const void* a, const void* b, int64_t numel,
                   void* out, void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    if (mode == CSD_MODE_PROD) return set_error(CSD_ERR_UNSUPPORTED, "csd_add: CHECK mode only");
    CSD_CU(check_add((const float*)a, (const float*)b, numel, (float*)out, S(stream)), "add");
    c->launches += 1;
    return CSD_OK;
}

}  // extern "C"

extern "C" {

csd_status csd_mlp_preact(csd_ctx* ctx, csd_mode mode, const void* x, const void* w1,
                          const float* b1, int64_t batch, int64_t n, int64_t d, int64_t f,
                          float* pre_out, void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    CSD_TRY(check_mlp_shape(batch, n, d, f));
    if (mode != CSD_MODE_CHECK)
        return set_error(CSD_ERR_UNSUPPORTED, "csd_mlp_preact: CHECK mode only");
    CSD_CU(check_mlp_preact((const float*)x, (const float*)w1, b1, batch * n, d, f, pre_out,
                            S(stream)), "mlp_preact");
    c->launches += 1;
    return CSD_OK;
}

csd_status csd_device_alloc(size_t bytes, void** out) {
    if (!out) return set_error(CSD_ERR_VALUE, "csd_device_alloc: null out");
    *out = nullptr;
    CSD_CU(cudaMalloc(out, bytes ? bytes : 16), "cudaMalloc");
    return CSD_OK;
}
csd_status csd_device_free(void* ptr) {
    if (ptr) CSD_CU(cudaFree(ptr), "cudaFree");
    return CSD_OK;
}
csd_status csd_copy_to_device(void* dst, const void* src, size_t bytes) {
    if (bytes) CSD_CU(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "cudaMemcpy h2d");
    return CSD_OK;
}
csd_status csd_copy_to_host(void* dst, const void* src, size_t bytes) {
    if (bytes) CSD_CU(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), "cudaMemcpy d2h");
    return CSD_OK;
}
csd_status csd_cast(csd_ctx* ctx, const void* src, void* dst, int64_t n, int to_bf16, void* stream) {
    auto* c = reinterpret_cast<Ctx*>(ctx);
    if (!c || (n > 0 && (!src || !dst))) return set_error(CSD_ERR_VALUE, "csd_cast: null argument");
    if (n < 0) return set_error(CSD_ERR_VALUE, "csd_cast: negative count");
    if (to_bf16)
        CSD_CU(prod_cast_f32_bf16(static_cast<const float*>(src), dst, n, S(stream)), "cast");
    else
        CSD_CU(prod_cast_bf16_f32(src, static_cast<float*>(dst), n, S(stream)), "cast");
    c->launches += 1;
    return CSD_OK;
}

}  // extern "C"
