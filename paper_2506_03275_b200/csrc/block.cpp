// block.cpp — device-resident DiT block (model_forward_step for one layer,
// model.cpp:178-216) behind csd_block_*.
//
//   q,k,v = x Wq, x Wk, x Wv                 (token-major [B,N,H*E]: no split_heads)
//   dense : O, m, l, colsum = column_sum_attention(q,k,v, stale m,l)   (attention.cpp:202-215)
//           idx = top-k(colsum) | static pattern;  resid = O - sparse(idx)
//   sparse: O = resid + sparse(idx)                                     (attention.cpp:217-218)
//   x1 = x + O Wo
//   dense : M = dense_mlp(x1), A = act, T_m = tile_means(x1)             (mlp.cpp:196-205)
//   sparse: S = top-k |tile_means(x1) - T_m|;  A, M updated by the delta (mlp.cpp:206-210)
//   x2 = x1 + M
// CHECK mode runs every op on the bit-exact kernels (fp32); PROD mode keeps
// activations in bf16, caches in bf16/fp32, and uses the tcgen05 attention.
#include <cstring>
#include <vector>

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

struct csd_block {
    Ctx* ctx = nullptr;
    csd_mode mode = CSD_MODE_CHECK;
    csd_block_config cfg{};
    std::vector<void*> allocs;
    // weights
    void *wq = nullptr, *wk = nullptr, *wv = nullptr, *wo = nullptr, *w1 = nullptr, *w2 = nullptr;
    float *b1 = nullptr, *b2 = nullptr;
    // activations
    void *q = nullptr, *k = nullptr, *v = nullptr, *attn = nullptr, *x_mid = nullptr;
    float* proj = nullptr;  // [B,N,D] fp32 branch output
    // caches
    void* resid = nullptr;
    float *m[2] = {nullptr, nullptr}, *l[2] = {nullptr, nullptr};
    int cur = 0;
    float* colsum = nullptr;
    int32_t *aidx = nullptr, *acnt = nullptr;
    int64_t a_kmax = 0;
    float* tmeans = nullptr;
    void* act = nullptr;
    float* mout = nullptr;
    int32_t *midx = nullptr, *mcnt = nullptr;
    bool attn_init = false, mlp_init = false;
    // scratch of the cache-free dense forward (CSD_BLOCK_FORWARD_DENSE), allocated on first use
    void* plain_act = nullptr;
    float* plain_mout = nullptr;
    int64_t attn_age = 0, mlp_age = 0;
    // the MLP's view of the rows: (batch, seq) of the block, or (1, t_local) when token-sharded
    int64_t mB = 0, mN = 0;
    bool token_mode = false;

    // The persistent caches (everything a later step reads: attention residual, stats, index
    // sets, MLP activations / outputs / tile means) live in ONE arena, so a layer stack can
    // keep two arenas on the device and stream the others to host memory (memory.cpp:33-58,
    // "optimized double-buffers two layers while the rest live off-device";
    // csd_block_bind_cache_arena).  Per-step scratch stays in `allocs`.
    void* arena = nullptr;
    bool arena_owned = true;
    size_t arena_bytes = 0;
    std::vector<std::pair<void**, size_t>> arena_slots;  // (pointer field, offset)

    void* alloc(size_t bytes) {
        void* p = nullptr;
        if (cudaMalloc(&p, bytes < 256 ? 256 : bytes) != cudaSuccess) return nullptr;
        allocs.push_back(p);
        return p;
    }
    // reserve `bytes` of the cache arena for *field (bound by finish_arena)
    void cache_alloc(void** field, size_t bytes) {
        arena_slots.emplace_back(field, arena_bytes);
        arena_bytes += (bytes + 255) & ~size_t(255);
    }
    bool bind_arena(void* base) {
        for (auto& sl : arena_slots) *sl.first = static_cast<char*>(base) + sl.second;
        arena = base;
        return true;
    }
    bool finish_arena() {
        if (cudaMalloc(&arena, arena_bytes < 256 ? 256 : arena_bytes) != cudaSuccess) {
            arena = nullptr;
            return false;
        }
        arena_owned = true;
        return bind_arena(arena);
    }
    ~csd_block() {
        for (void* p : allocs) cudaFree(p);
        if (arena_owned && arena) cudaFree(arena);
    }
};

namespace {

size_t esz(csd_mode m) { return m == CSD_MODE_PROD ? 2 : 4; }

// Upload a host fp32 sub-matrix (rows r0.., cols c0..) in the mode's dtype.
csd_status upload(csd_block* blk, void** dst, const float* host, int64_t rows, int64_t cols,
                  int64_t ld, int64_t r0, int64_t c0, bool keep_f32) {
    const size_t n = (size_t)(rows * cols);
    std::vector<float> tmp(n);
    for (int64_t r = 0; r < rows; ++r)
        std::memcpy(&tmp[r * cols], host + (r0 + r) * ld + c0, sizeof(float) * cols);
    const bool bf = blk->mode == CSD_MODE_PROD && !keep_f32;
    void* d = blk->alloc(n * (bf ? 2 : 4));
    if (!d) return set_error(CSD_ERR_CUDA, "block weight allocation failed");
    if (bf) {
        float* staging = nullptr;
        CSD_CU(cudaMalloc(&staging, n * 4), "cudaMalloc");
        CSD_CU(cudaMemcpy(staging, tmp.data(), n * 4, cudaMemcpyHostToDevice), "h2d");
        CSD_CU(prod_cast_f32_bf16(staging, d, (int64_t)n, nullptr), "cast");
        CSD_CU(cudaDeviceSynchronize(), "sync");
        cudaFree(staging);
    } else {
        CSD_CU(cudaMemcpy(d, tmp.data(), n * 4, cudaMemcpyHostToDevice), "h2d");
    }
    *dst = d;
    return CSD_OK;
}

}  // namespace

static csd_status attn_core(csd_block* blk, const void* x_in, int dense, const int32_t* static_idx,
                            const int32_t* static_counts, int64_t static_k_max, void* stream);
static csd_ctx* ctx_of(csd_block* blk) { return reinterpret_cast<csd_ctx*>(blk->ctx); }
static csd_status sparse_mlp_apply(csd_block* blk, const void* x_mid, void* x_out, cudaStream_t s);

extern "C" {

csd_status csd_block_create(csd_ctx* ctx, csd_mode mode, const csd_block_config* cfg_in,
                            const float* wq, const float* wk, const float* wv, const float* wo,
                            const float* w1, const float* b1, const float* w2, const float* b2,
                            csd_block** out) {
    if (!ctx || !cfg_in || !out) return set_error(CSD_ERR_VALUE, "csd_block_create: null argument");
    csd_block_config c = *cfg_in;
    if (c.heads_local == 0) c.heads_local = c.heads;
    if (c.f_local == 0) c.f_local = c.hidden;
    // model.cpp:10-28 validation
    if (c.batch < 1 || c.seq < 1 || c.dim < 1 || c.heads < 1 || c.head_dim < 1 || c.hidden < 1 ||
        c.chunk < 1)
        return set_error(CSD_ERR_CONFIG, "model config fields must be positive");
    if (c.dim != c.heads * c.head_dim)
        return set_error(CSD_ERR_CONFIG, "model_dim %lld != heads*head_dim %lld", (long long)c.dim,
                         (long long)(c.heads * c.head_dim));
    if (c.seq % c.chunk)
        return set_error(CSD_ERR_CONFIG, "sequence length %lld not divisible by chunk %lld",
                         (long long)c.seq, (long long)c.chunk);
    if (c.head0 < 0 || c.head0 + c.heads_local > c.heads || c.f0 < 0 || c.f0 + c.f_local > c.hidden)
        return set_error(CSD_ERR_CONFIG, "shard outside the block");
    const bool token_mode = c.t_local > 0;
    if (token_mode) {
        // token rows are whole chunks (chunks never straddle sequences: seq % chunk == 0)
        if (mode != CSD_MODE_PROD)
            return set_error(CSD_ERR_UNSUPPORTED, "token-sharded blocks are PROD only");
        if (c.t0 < 0 || c.t0 % c.chunk || c.t_local % c.chunk || c.t0 + c.t_local > c.batch * c.seq)
            return set_error(CSD_ERR_CONFIG, "token rows [%lld, +%lld) not chunk-aligned inside the block",
                             (long long)c.t0, (long long)c.t_local);
        if (c.f0 != 0 || c.f_local != c.hidden)
            return set_error(CSD_ERR_CONFIG, "token-sharded blocks keep every hidden neuron");
    }
    auto* blk = new csd_block;
    blk->ctx = reinterpret_cast<Ctx*>(ctx);
    blk->mode = mode;
    blk->cfg = c;
    const int64_t B = c.batch, N = c.seq, D = c.dim, E = c.head_dim, Hl = c.heads_local;
    const int64_t Dl = Hl * E, Fl = c.f_local, C = N / c.chunk;
    csd_status st = CSD_OK;
    auto fail = [&](csd_status s) {
        delete blk;
        return s;
    };
    const int64_t col0 = c.head0 * E;
    if ((st = upload(blk, &blk->wq, wq, D, Dl, D, 0, col0, false)) != CSD_OK) return fail(st);
    if ((st = upload(blk, &blk->wk, wk, D, Dl, D, 0, col0, false)) != CSD_OK) return fail(st);
    if ((st = upload(blk, &blk->wv, wv, D, Dl, D, 0, col0, false)) != CSD_OK) return fail(st);
    // output projection: this shard's head rows of Wo, or all of it for token rows
    if ((st = upload(blk, &blk->wo, wo, token_mode ? D : Dl, D, D, token_mode ? 0 : col0, 0, false)) != CSD_OK)
        return fail(st);
    if ((st = upload(blk, &blk->w1, w1, Fl, D, D, c.f0, 0, false)) != CSD_OK) return fail(st);
    if ((st = upload(blk, &blk->w2, w2, Fl, D, D, c.f0, 0, false)) != CSD_OK) return fail(st);
    void* tmp = nullptr;
    if ((st = upload(blk, &tmp, b1, 1, Fl, Fl, 0, c.f0, true)) != CSD_OK) return fail(st);
    blk->b1 = (float*)tmp;
    std::vector<float> b2l(D, 0.0f);
    if (c.f0 == 0) std::memcpy(b2l.data(), b2, sizeof(float) * D);  // bias once across shards
    if ((st = upload(blk, &tmp, b2l.data(), 1, D, D, 0, 0, true)) != CSD_OK) return fail(st);
    blk->b2 = (float*)tmp;

    blk->token_mode = token_mode;
    blk->mB = token_mode ? 1 : B;
    blk->mN = token_mode ? c.t_local : N;
    const int64_t MR = blk->mB * blk->mN, MC = MR / c.chunk;  // MLP rows / chunks
    const size_t es = esz(mode);
    // per-step scratch
    blk->q = blk->alloc(es * B * N * Dl);
    blk->k = blk->alloc(es * B * N * Dl);
    blk->v = blk->alloc(es * B * N * Dl);
    blk->attn = blk->alloc(es * B * N * Dl);
    blk->x_mid = blk->alloc(es * (token_mode ? MR : B * N) * D);
    blk->proj = (float*)blk->alloc(4 * B * N * D);
    blk->colsum = (float*)blk->alloc(4 * B * Hl * C * N);
    // persistent caches: one arena
    const int64_t ak = c.attn_k > 0 ? c.attn_k : N;
    const int64_t mk = c.mlp_k > 0 ? c.mlp_k : Fl;
    blk->a_kmax = ak;
    blk->cache_alloc(&blk->resid, es * B * N * Dl);
    for (int i = 0; i < 2; ++i) {
        blk->cache_alloc(reinterpret_cast<void**>(&blk->m[i]), 4 * B * Hl * N);
        blk->cache_alloc(reinterpret_cast<void**>(&blk->l[i]), 4 * B * Hl * N);
    }
    blk->cache_alloc(reinterpret_cast<void**>(&blk->aidx), 4 * B * Hl * C * ak);
    blk->cache_alloc(reinterpret_cast<void**>(&blk->acnt), 4 * B * Hl * C);
    blk->cache_alloc(reinterpret_cast<void**>(&blk->tmeans), 4 * MC * Fl);
    blk->cache_alloc(&blk->act, es * MR * Fl);
    blk->cache_alloc(reinterpret_cast<void**>(&blk->mout), 4 * MR * D);
    blk->cache_alloc(reinterpret_cast<void**>(&blk->midx), 4 * MC * mk);
    blk->cache_alloc(reinterpret_cast<void**>(&blk->mcnt), 4 * MC);
    for (void* p : blk->allocs)
        if (!p) return fail(set_error(CSD_ERR_CUDA, "block allocation failed"));
    if (!blk->finish_arena()) return fail(set_error(CSD_ERR_CUDA, "block cache arena allocation failed"));
    *out = blk;
    return CSD_OK;
}

csd_status csd_block_reset(csd_block* blk) {
    // make_state (model.cpp:101-105): every cache empty again, so the next step must be
    // dense and sees no stale softmax stats (fresh ones, attention.cpp:122-137)
    if (!blk) return set_error(CSD_ERR_VALUE, "null block");
    blk->attn_init = blk->mlp_init = false;
    blk->attn_age = blk->mlp_age = 0;
    blk->cur = 0;
    return CSD_OK;
}

csd_status csd_block_cache_arena(csd_block* blk, void** dev_ptr, size_t* bytes) {
    if (!blk) return set_error(CSD_ERR_VALUE, "null block");
    if (dev_ptr) *dev_ptr = blk->arena;
    if (bytes) *bytes = blk->arena_bytes;
    return CSD_OK;
}

csd_status csd_block_bind_cache_arena(csd_block* blk, void* dev_ptr, size_t bytes) {
    // Re-point the block's caches into caller storage of >= csd_block_cache_arena bytes (the
    // same layout); the block's own arena is released.  The contents are NOT copied: the caller
    // moves them (a layer stack streams each layer's arena between host memory and two device
    // slots).  CUDA graphs captured before a rebind keep the old addresses.
    if (!blk || !dev_ptr) return set_error(CSD_ERR_VALUE, "null block or arena");
    if (bytes < blk->arena_bytes)
        return set_error(CSD_ERR_SHAPE, "cache arena of %zu bytes < the block's %zu", bytes, blk->arena_bytes);
    if (reinterpret_cast<uintptr_t>(dev_ptr) % 256 != 0)
        return set_error(CSD_ERR_VALUE, "cache arena must be 256-byte aligned");
    if (blk->arena_owned && blk->arena && blk->arena != dev_ptr) {
        cudaDeviceSynchronize();
        cudaFree(blk->arena);
    }
    blk->arena_owned = false;
    blk->bind_arena(dev_ptr);
    return CSD_OK;
}

csd_status csd_block_destroy(csd_block* blk) {
    cudaDeviceSynchronize();
    delete blk;
    return CSD_OK;
}

csd_status csd_block_step(csd_block* blk, const void* x_in, void* x_out, int dense,
                          const int32_t* static_idx, const int32_t* static_counts,
                          int64_t static_k_max, void* stream) {
    if (!blk) return set_error(CSD_ERR_VALUE, "null block");
    if (blk->token_mode)
        return set_error(CSD_ERR_UNSUPPORTED, "token-sharded block: use csd_block_attn_heads / csd_block_rows_step");
    const auto& c = blk->cfg;
    csd_ctx* ctx = reinterpret_cast<csd_ctx*>(blk->ctx);
    const csd_mode md = blk->mode;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (dense < 0 || dense > 2) return set_error(CSD_ERR_VALUE, "step kind %d (0 sparse, 1 dense, 2 forward-dense)", dense);
    const bool plain = dense == 2;
    if (!dense && (!blk->attn_init || !blk->mlp_init))
        return set_error(CSD_ERR_STATE, "sparse attention step requested before any dense step");
    if (plain && static_idx)
        return set_error(CSD_ERR_VALUE, "the cache-free dense forward takes no attention pattern");
    if (plain && !blk->plain_act) {  // first use (eager, before any graph capture of it)
        blk->plain_act = blk->alloc(esz(md) * c.batch * c.seq * c.f_local);
        blk->plain_mout = static_cast<float*>(blk->alloc(4 * c.batch * c.seq * c.dim));
        if (!blk->plain_act || !blk->plain_mout) return set_error(CSD_ERR_CUDA, "forward-dense scratch allocation failed");
    }
    void* const act = plain ? blk->plain_act : blk->act;
    float* const mout = plain ? blk->plain_mout : blk->mout;
    if (dense && static_idx) {
        // A caller-supplied static pattern (attention.cpp:205-213) is checked BEFORE anything
        // runs, so a bad pattern leaves every cache untouched (as the reference, which throws
        // before mutating the AttentionCache): k_max must be the block's, ids in [0, N)
        // without duplicates, counts in [0, k_max].  Synchronous unless the stream is being
        // captured (then the device flags surface at csd_ctx_sync).
        if (!static_counts)
            return set_error(CSD_ERR_VALUE, "static attention pattern without counts");
        if (static_k_max != blk->a_kmax)
            return set_error(CSD_ERR_SHAPE, "static pattern k_max %lld != block attn_k %lld",
                             (long long)static_k_max, (long long)blk->a_kmax);
        const cudaStream_t vs = static_cast<cudaStream_t>(stream);
        const int64_t rows = c.batch * c.heads_local * (c.seq / c.chunk);
        CSD_TRY(csd_validate_index_set(ctx_of(blk), static_idx, static_counts, rows, static_k_max,
                                       c.seq, stream));
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(vs, &cs) != cudaSuccess || cs == cudaStreamCaptureStatusNone)
            CSD_TRY(csd::check_flags(blk->ctx, vs));
    }
    // PROD: the selected index sets feed order-invariant kernels -> skip the per-row sort
    struct SortGuard {
        Ctx* c;
        bool old;
        ~SortGuard() { c->sorted_topk = old; }
    } sort_guard{blk->ctx, blk->ctx->sorted_topk};
    blk->ctx->sorted_topk = md != CSD_MODE_PROD;
    const int64_t B = c.batch, N = c.seq, D = c.dim;
    const int64_t Dl = c.heads_local * c.head_dim, Fl = c.f_local;
    const int64_t mk = c.mlp_k > 0 ? c.mlp_k : Fl;
    CSD_TRY(attn_core(blk, x_in, dense, static_idx, static_counts, static_k_max, stream));
    if (md == CSD_MODE_PROD) {
        // x1 = x + O Wo: the residual rides in the GEMM epilogue (gemm_tc.cu); the library
        // fallback adds it as C = x, beta = 1 over a copy
        if (csd::dev::gemm_tc_enabled() && csd::dev::gemm_tc_proj_supported(B * N, Dl, D)) {
            const void* w[3] = {blk->wo, blk->wo, blk->wo};
            void* o[3] = {blk->x_mid, blk->x_mid, blk->x_mid};
            CSD_CU(csd::dev::gemm_tc_proj(blk->attn, w, o, 1, B * N, Dl, D, x_in, s), "gemm_tc_wo");
            blk->ctx->launches += 1;
        } else {
            CSD_CU(cudaMemcpyAsync(blk->x_mid, x_in, 2 * B * N * D, cudaMemcpyDeviceToDevice, s), "copy");
            CSD_TRY(csd::gemm_bf16(blk->ctx, blk->attn, blk->wo, false, blk->x_mid, false, B * N, D,
                                   Dl, 1.0f, s));
        }
        // ---- MLP branch; x2 = x1 + M is fused into the last MLP kernel's epilogue.  With
        // mlp_k >= F every neuron is recomputed on a sparse step (mlp.cpp:120-182 with the full
        // index set), which is the dense MLP with the cache refreshed (WAN-style configs)
        if (plain) {  // dense MLP into scratch: the caches stay as the last dense step left them
            CSD_TRY(csd::prod_dense_mlp(blk->ctx, blk->x_mid, blk->w1, blk->b1, blk->w2, blk->b2, B,
                                        N, D, Fl, c.chunk, mout, act, blk->x_mid, x_out, s));
            return CSD_OK;
        }
        if (dense || mk >= Fl) {
            CSD_TRY(csd::prod_dense_mlp(blk->ctx, blk->x_mid, blk->w1, blk->b1, blk->w2, blk->b2, B,
                                        N, D, Fl, c.chunk, blk->mout, blk->act, blk->x_mid, x_out,
                                        s));
            if (dense)  // the selection signal (unused when every neuron is recomputed)
                CSD_TRY(csd_mlp_tile_means(ctx, md, blk->x_mid, blk->w1, B, N, D, Fl, c.chunk,
                                           blk->tmeans, stream));
            blk->mlp_init = true;
            blk->mlp_age = dense ? 0 : blk->mlp_age + 1;
        } else {
            CSD_TRY(csd_mlp_change_indices(ctx, md, blk->x_mid, blk->w1, blk->tmeans, B, N, D, Fl,
                                           mk, c.chunk, blk->midx, blk->mcnt, stream));
            CSD_TRY(sparse_mlp_apply(blk, blk->x_mid, x_out, s));
        }
        return CSD_OK;
    }
    // ---------------- CHECK mode: op for op as model.cpp:200-213
    CSD_TRY(csd_project(ctx, md, blk->attn, blk->wo, B, N, Dl, D, blk->proj, stream));
    CSD_TRY(csd_add(ctx, md, x_in, blk->proj, B * N * D, blk->x_mid, stream));
    if (plain) {
        CSD_TRY(csd_dense_mlp(ctx, md, blk->x_mid, blk->w1, blk->b1, blk->w2, blk->b2, B, N, D, Fl,
                              c.chunk, mout, act, stream));
        return csd_add(ctx, md, blk->x_mid, mout, B * N * D, x_out, stream);
    }
    if (dense) {
        CSD_TRY(csd_dense_mlp(ctx, md, blk->x_mid, blk->w1, blk->b1, blk->w2, blk->b2, B, N, D, Fl,
                              c.chunk, blk->mout, blk->act, stream));
        CSD_TRY(csd_mlp_tile_means(ctx, md, blk->x_mid, blk->w1, B, N, D, Fl, c.chunk, blk->tmeans,
                                   stream));
        blk->mlp_init = true;
        blk->mlp_age = 0;
    } else {
        CSD_TRY(csd_mlp_change_indices(ctx, md, blk->x_mid, blk->w1, blk->tmeans, B, N, D, Fl, mk,
                                       c.chunk, blk->midx, blk->mcnt, stream));
        CSD_TRY(csd_sparse_delta_mlp(ctx, md, blk->x_mid, blk->w1, blk->b1, blk->w2, blk->midx,
                                     blk->mcnt, mk, c.chunk, B, N, D, Fl, blk->act, blk->mout,
                                     stream));
        blk->mlp_age += 1;
    }
    CSD_TRY(csd_add(ctx, md, blk->x_mid, blk->mout, B * N * D, x_out, stream));
    return CSD_OK;
}

}  // extern "C"

// ---- attention branch of a step (shared by the whole-block and the sharded paths):
// q,k,v for the block's heads, then colsum/top-k/cache-init (dense) or the sparse delta.
static csd_status attn_core(csd_block* blk, const void* x_in, int dense, const int32_t* static_idx,
                            const int32_t* static_counts, int64_t static_k_max, void* stream) {
    const auto& c = blk->cfg;
    csd_ctx* ctx = reinterpret_cast<csd_ctx*>(blk->ctx);
    const csd_mode md = blk->mode;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t B = c.batch, N = c.seq, D = c.dim, E = c.head_dim, Hl = c.heads_local;
    const int64_t Dl = Hl * E, C = N / c.chunk;
    const int64_t ak = blk->a_kmax;
    if (md == CSD_MODE_PROD && csd::dev::gemm_tc_enabled() &&
        csd::dev::gemm_tc_proj_supported(B * N, D, Dl)) {
        // one tcgen05 launch for the three projections (gemm_tc.cu), bf16 [B, N, H, E] out
        const void* w[3] = {blk->wq, blk->wk, blk->wv};
        void* o[3] = {blk->q, blk->k, blk->v};
        CSD_CU(csd::dev::gemm_tc_proj(x_in, w, o, 3, B * N, D, Dl, nullptr, s), "gemm_tc_qkv");
        blk->ctx->launches += 1;
    } else {
        CSD_TRY(csd_project(ctx, md, x_in, blk->wq, B, N, D, Dl, blk->q, stream));
        CSD_TRY(csd_project(ctx, md, x_in, blk->wk, B, N, D, Dl, blk->k, stream));
        CSD_TRY(csd_project(ctx, md, x_in, blk->wv, B, N, D, Dl, blk->v, stream));
    }
    if (dense == 2) {  // model_forward_dense (model.cpp:167-176): exact attention, no caches
        return csd_dense_attention(ctx, md, CSD_LAYOUT_BNHE, blk->q, blk->k, blk->v, B, Hl, N, E,
                                   blk->attn, stream);
    }
    // Index sets produced inside the block are valid by construction (top-k); a static
    // pattern was validated by csd_block_step before anything ran.  Skip per-call validation.
    struct ValidateGuard {
        Ctx* c;
        bool old;
        ~ValidateGuard() { c->validate_prod = old; }
    } vguard{blk->ctx, blk->ctx->validate_prod};
    blk->ctx->validate_prod = false;
    // the block's own top-k sets have count k in every chunk: nothing for LPT to balance;
    // a caller's static pattern is ragged
    struct LptGuard {
        Ctx* c;
        bool old;
        ~LptGuard() { c->lpt = old; }
    } lguard{blk->ctx, blk->ctx->lpt};
    blk->ctx->lpt = static_idx != nullptr;
    if (dense) {
        // PROD reads the stale stats and writes the fresh ones row-by-row in the
        // same thread, so one buffer suffices (and the step stays graph-capturable);
        // CHECK mode's colsum pass re-reads the stats after softmax -> double buffer.
        const int nxt = (blk->attn_init && md == CSD_MODE_CHECK) ? 1 - blk->cur : blk->cur;
        const float* pm = blk->attn_init ? blk->m[blk->cur] : nullptr;
        const float* pl = blk->attn_init ? blk->l[blk->cur] : nullptr;
        CSD_TRY(csd_column_sum_attention(ctx, md, CSD_LAYOUT_BNHE, blk->q, blk->k, blk->v, pm, pl, B,
                                         Hl, N, E, c.chunk, blk->attn, blk->m[nxt], blk->l[nxt],
                                         blk->colsum, stream));
        blk->cur = nxt;
        const int32_t* ui = blk->aidx;
        const int32_t* uc = blk->acnt;
        int64_t ukm = ak;
        if (static_idx) {
            ui = static_idx;
            uc = static_counts;
            ukm = static_k_max;
        } else {
            CSD_TRY(csd_select_top_k(ctx, blk->colsum, B * Hl * C, N, ak, blk->aidx, blk->acnt,
                                     stream));
        }
        if (static_idx) {  // keep a private copy (the cache owns its indices)
            CSD_CU(cudaMemcpyAsync(blk->aidx, static_idx, 4 * B * Hl * C * ukm,
                                   cudaMemcpyDeviceToDevice, s), "copy");
            CSD_CU(cudaMemcpyAsync(blk->acnt, static_counts, 4 * B * Hl * C,
                                   cudaMemcpyDeviceToDevice, s), "copy");
        }
        (void)ui;
        (void)uc;
        CSD_TRY(csd_sparse_delta_attention(ctx, md, CSD_LAYOUT_BNHE, blk->q, blk->k, blk->v,
                                           blk->aidx, blk->acnt, ukm, c.chunk, blk->attn, -1.0f,
                                           B, Hl, N, E, blk->resid, stream));
        blk->attn_init = true;
        blk->attn_age = 0;
    } else {
        CSD_TRY(csd_sparse_delta_attention(ctx, md, CSD_LAYOUT_BNHE, blk->q, blk->k, blk->v,
                                           blk->aidx, blk->acnt, ak, c.chunk, blk->resid, 1.0f, B,
                                           Hl, N, E, blk->attn, stream));
        blk->attn_age += 1;
    }
    return CSD_OK;
}

// ---- PROD sparse-delta MLP with the block's current index set (midx / mcnt); optional
// fused residual x_out = x_mid + M_cache.
static csd_status sparse_mlp_apply(csd_block* blk, const void* x_mid, void* x_out, cudaStream_t s) {
    const auto& c = blk->cfg;
    const int64_t B = blk->mB, N = blk->mN, D = c.dim, Fl = c.f_local;
    const int64_t mk = c.mlp_k > 0 ? c.mlp_k : Fl;
    if (!mlp_tc_supported(D, c.chunk))
        return set_error(CSD_ERR_UNSUPPORTED, "sparse-delta MLP envelope (D %% 128, chunk <= 256)");
    const int64_t k_pad = csd::dev::prod_smlp_delta_cols(mk, B * (N / c.chunk), c.chunk);
    void* dws = blk->ctx->ws(csd::kWsDelta, 2 * B * N * k_pad, s);
    if (!dws) return set_error(CSD_ERR_CUDA, "workspace allocation failed");
    CSD_CU(prod_sparse_delta_mlp_tc(x_mid, blk->w1, blk->b1, blk->w2, blk->midx, blk->mcnt, mk,
                                    c.chunk, B, N, D, Fl, blk->act, blk->mout, dws, s, x_mid, x_out),
           "sparse_delta_mlp");
    blk->ctx->launches += 2;
    blk->mlp_age += 1;
    return CSD_OK;
}

extern "C" {

// ---------------------------------------------------------------- sharded execution
csd_status csd_block_attn_partial(csd_block* blk, const void* x_in, int dense,
                                  float* attn_partial, void* stream) {
    if (!blk) return set_error(CSD_ERR_VALUE, "null block");
    if (blk->mode != CSD_MODE_PROD) return set_error(CSD_ERR_UNSUPPORTED, "sharded steps are PROD only");
    if (!dense && !blk->attn_init)
        return set_error(CSD_ERR_STATE, "sparse attention step requested before any dense step");
    const auto& c = blk->cfg;
    CSD_TRY(attn_core(blk, x_in, dense, nullptr, nullptr, 0, stream));
    // this rank's heads through its rows of Wo: a partial [B, N, D] sum (all-reduced by the caller)
    return csd::gemm_bf16(blk->ctx, blk->attn, blk->wo, false, attn_partial, true, c.batch * c.seq,
                          c.dim, c.heads_local * c.head_dim, 0.0f, static_cast<cudaStream_t>(stream));
}

csd_status csd_block_mlp_dense_partial(csd_block* blk, const void* x_mid, float* mlp_partial,
                                       void* stream) {
    if (!blk) return set_error(CSD_ERR_VALUE, "null block");
    if (blk->mode != CSD_MODE_PROD) return set_error(CSD_ERR_UNSUPPORTED, "sharded steps are PROD only");
    const auto& c = blk->cfg;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t B = c.batch, N = c.seq, D = c.dim, Fl = c.f_local;
    CSD_TRY(csd::prod_dense_mlp(blk->ctx, x_mid, blk->w1, blk->b1, blk->w2, blk->b2, B, N, D, Fl,
                                c.chunk, blk->mout, blk->act, nullptr, nullptr, s));
    CSD_TRY(csd_mlp_tile_means(reinterpret_cast<csd_ctx*>(blk->ctx), blk->mode, x_mid, blk->w1, B, N,
                               D, Fl, c.chunk, blk->tmeans, stream));
    CSD_CU(cudaMemcpyAsync(mlp_partial, blk->mout, 4 * B * N * D, cudaMemcpyDeviceToDevice, s), "copy");
    blk->mlp_init = true;
    blk->mlp_age = 0;
    return CSD_OK;
}

csd_status csd_block_mlp_candidates(csd_block* blk, const void* x_mid, float* cand_scores,
                                    int32_t* cand_ids, void* stream) {
    if (!blk) return set_error(CSD_ERR_VALUE, "null block");
    if (blk->mode != CSD_MODE_PROD) return set_error(CSD_ERR_UNSUPPORTED, "sharded steps are PROD only");
    if (!blk->mlp_init) return set_error(CSD_ERR_STATE, "sparse MLP step requested before any dense step");
    const auto& c = blk->cfg;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t B = c.batch, N = c.seq, D = c.dim, Fl = c.f_local, rows = B * (N / c.chunk);
    const int64_t k = c.mlp_k > 0 ? c.mlp_k : c.hidden;
    const int64_t k_loc = k < Fl ? k : Fl;
    float* scores = (float*)blk->ctx->ws(csd::kWsScores, 4 * rows * Fl, s);
    void* ws = blk->ctx->ws(csd::kWsMeans, prod_means_ws_bytes(B, N, D, Fl, c.chunk), s);
    int32_t* ids = (int32_t*)blk->ctx->ws(csd::kWsIdx, 4 * rows * k_loc, s);
    int32_t* cnt = (int32_t*)blk->ctx->ws(csd::kWsCounts, 4 * rows, s);
    if (!scores || !ws || !ids || !cnt) return set_error(CSD_ERR_CUDA, "workspace allocation failed");
    // local |T - T_m| (mlp.cpp:116) and the shard's top-k
    CSD_CU(prod_tile_means_tc(x_mid, blk->w1, B, N, D, Fl, c.chunk, blk->tmeans, scores, ws, s),
           "tile_means");
    CSD_CU(topk_rows(scores, rows, Fl, k_loc, ids, cnt, s), "topk");
    CSD_CU(shard_candidates(ids, scores, rows, Fl, k_loc, k, c.f0, cand_scores, cand_ids, s),
           "candidates");
    blk->ctx->launches += 5;
    return CSD_OK;
}

csd_status csd_block_mlp_sparse_partial(csd_block* blk, const void* x_mid,
                                        const float* all_scores, const int32_t* all_ids,
                                        int64_t world, float* mlp_partial, void* stream) {
    if (!blk) return set_error(CSD_ERR_VALUE, "null block");
    if (blk->mode != CSD_MODE_PROD) return set_error(CSD_ERR_UNSUPPORTED, "sharded steps are PROD only");
    if (!blk->mlp_init) return set_error(CSD_ERR_STATE, "sparse MLP step requested before any dense step");
    if (world < 1) return set_error(CSD_ERR_VALUE, "world size must be >= 1");
    const auto& c = blk->cfg;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t B = c.batch, N = c.seq, D = c.dim, rows = B * (N / c.chunk);
    const int64_t k = c.mlp_k > 0 ? c.mlp_k : c.hidden;
    float* ws_s = (float*)blk->ctx->ws(csd::kWsLogits, 4 * rows * world * k, s);
    int32_t* ws_i = (int32_t*)blk->ctx->ws(csd::kWsProbs, 4 * rows * world * k, s);
    int32_t* ws_p = (int32_t*)blk->ctx->ws(csd::kWsIdx, 4 * rows * k, s);
    int32_t* ws_c = (int32_t*)blk->ctx->ws(csd::kWsCounts, 4 * rows, s);
    if (!ws_s || !ws_i || !ws_p || !ws_c) return set_error(CSD_ERR_CUDA, "workspace allocation failed");
    const int64_t mk = c.mlp_k > 0 ? c.mlp_k : c.f_local;  // row stride of midx
    CSD_CU(shard_merge(all_scores, all_ids, world, rows, k, c.f0, c.f_local, ws_s, ws_i, ws_p, ws_c,
                       blk->midx, mk, blk->mcnt, s),
           "merge");
    blk->ctx->launches += 3;
    CSD_TRY(sparse_mlp_apply(blk, x_mid, nullptr, s));
    CSD_CU(cudaMemcpyAsync(mlp_partial, blk->mout, 4 * B * N * D, cudaMemcpyDeviceToDevice, s), "copy");
    return CSD_OK;
}

// ---------------------------------------------------------------- token-sharded execution
csd_status csd_block_attn_heads(csd_block* blk, const void* x_in, int dense, void* attn_local,
                                void* stream) {
    if (!blk || !x_in || !attn_local) return set_error(CSD_ERR_VALUE, "null argument");
    if (blk->mode != CSD_MODE_PROD) return set_error(CSD_ERR_UNSUPPORTED, "sharded steps are PROD only");
    if (!dense && !blk->attn_init)
        return set_error(CSD_ERR_STATE, "sparse attention step requested before any dense step");
    // the attention output lands in the caller's buffer (the block's attn buffer is not a cache)
    void* own = blk->attn;
    blk->attn = attn_local;
    const csd_status st = attn_core(blk, x_in, dense, nullptr, nullptr, 0, stream);
    blk->attn = own;
    return st;
}

csd_status csd_block_rows_step(csd_block* blk, const void* x_rows, const void* attn_rows,
                               int64_t world, int dense, void* x_out_rows, void* stream) {
    if (!blk || !x_rows || !attn_rows || !x_out_rows) return set_error(CSD_ERR_VALUE, "null argument");
    if (!blk->token_mode) return set_error(CSD_ERR_STATE, "block is not token-sharded (t_local == 0)");
    const auto& c = blk->cfg;
    const int64_t R = c.t_local, D = c.dim, Dl = c.heads_local * c.head_dim, Fl = c.f_local;
    if (world < 1 || world * Dl != D)
        return set_error(CSD_ERR_SHAPE, "token rows need equal head shards: world %lld x %lld != dim %lld",
                         (long long)world, (long long)Dl, (long long)D);
    if (!dense && !blk->mlp_init)
        return set_error(CSD_ERR_STATE, "sparse MLP step requested before any dense step");
    csd_ctx* ctx = reinterpret_cast<csd_ctx*>(blk->ctx);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t mk = c.mlp_k > 0 ? c.mlp_k : Fl;
    // x_mid = x + O Wo over the rank-blocked head outputs [world][R][Dl] (the all-to-all's
    // layout: the GEMM's A operand walks the blocks, no re-layout copy)
    if (!csd::dev::gemm_tc_enabled() || !csd::dev::gemm_tc_proj_supported(R, D, D) || Dl % 64)
        return set_error(CSD_ERR_UNSUPPORTED, "token rows: tcgen05 projection envelope (rows %% 128, dims %% 64)");
    CSD_CU(csd::dev::gemm_tc_proj_blocked(attn_rows, blk->wo, blk->x_mid, R, D, D, x_rows, Dl, R, s),
           "gemm_tc_wo_rows");
    blk->ctx->launches += 1;
    if (dense) {
        CSD_TRY(csd::prod_dense_mlp(blk->ctx, blk->x_mid, blk->w1, blk->b1, blk->w2, blk->b2, 1, R, D,
                                    Fl, c.chunk, blk->mout, blk->act, blk->x_mid, x_out_rows, s));
        CSD_TRY(csd_mlp_tile_means(ctx, blk->mode, blk->x_mid, blk->w1, 1, R, D, Fl, c.chunk,
                                   blk->tmeans, stream));
        blk->mlp_init = true;
        blk->mlp_age = 0;
    } else {
        CSD_TRY(csd_mlp_change_indices(ctx, blk->mode, blk->x_mid, blk->w1, blk->tmeans, 1, R, D, Fl,
                                       mk, c.chunk, blk->midx, blk->mcnt, stream));
        CSD_TRY(sparse_mlp_apply(blk, blk->x_mid, x_out_rows, s));
    }
    return CSD_OK;
}

csd_status csd_residual_add(csd_ctx* ctx, const void* x, const float* partial, int64_t numel,
                            void* out, void* stream) {
    CSD_CU(prod_add_bf16_f32(x, partial, numel, out, static_cast<cudaStream_t>(stream)), "add");
    reinterpret_cast<Ctx*>(ctx)->launches += 1;
    return CSD_OK;
}

csd_status csd_block_cache(csd_block* blk, int which, void* out, int32_t* counts_out,
                           void* stream) {
    if (!blk) return set_error(CSD_ERR_VALUE, "null block");
    const auto& c = blk->cfg;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t B = c.batch, N = c.seq, D = c.dim, E = c.head_dim, Hl = c.heads_local;
    const int64_t Fl = c.f_local, C = N / c.chunk;
    // the MLP caches cover the block's MLP rows (all of B x N, or the token shard's rows)
    const int64_t MB = blk->mB, MN = blk->mN, MC = MN / c.chunk;
    csd_ctx* ctx = reinterpret_cast<csd_ctx*>(blk->ctx);
    switch (which) {
        case 0: {  // residual [B,H,N,E] fp32 from token-major storage
            std::vector<char> dummy;
            const size_t es = esz(blk->mode);
            for (int64_t b = 0; b < B; ++b)
                for (int64_t h = 0; h < Hl; ++h) {
                    // strided 2D copy: N rows of E elements, src pitch Hl*E
                    const char* src = (const char*)blk->resid + ((b * N) * Hl + h) * E * es;
                    float* dst = (float*)out + ((b * Hl + h) * N) * E;
                    if (blk->mode == CSD_MODE_PROD) {
                        float* tmp = (float*)blk->ctx->ws(csd::kWsPre, 4 * N * Hl * E, s);
                        CSD_CU(prod_cast_bf16_f32((const char*)blk->resid + b * N * Hl * E * es, tmp,
                                                  N * Hl * E, s), "cast");
                        CSD_CU(cudaMemcpy2DAsync(dst, E * 4, tmp + h * E, Hl * E * 4, E * 4, N,
                                                 cudaMemcpyDeviceToDevice, s), "copy");
                    } else {
                        CSD_CU(cudaMemcpy2DAsync(dst, E * 4, src, Hl * E * 4, E * 4, N,
                                                 cudaMemcpyDeviceToDevice, s), "copy");
                    }
                }
            return CSD_OK;
        }
        case 1:
            CSD_CU(cudaMemcpyAsync(out, blk->m[blk->cur], 4 * B * Hl * N, cudaMemcpyDeviceToDevice, s), "copy");
            return CSD_OK;
        case 2:
            CSD_CU(cudaMemcpyAsync(out, blk->l[blk->cur], 4 * B * Hl * N, cudaMemcpyDeviceToDevice, s), "copy");
            return CSD_OK;
        case 3:
            return csd_mlp_act_cache_to_ref(ctx, blk->mode, blk->act, MB, MN, Fl, c.chunk, (float*)out,
                                            stream);
        case 4:
            CSD_CU(cudaMemcpyAsync(out, blk->mout, 4 * MB * MN * D, cudaMemcpyDeviceToDevice, s), "copy");
            return CSD_OK;
        case 5:
            CSD_CU(cudaMemcpyAsync(out, blk->tmeans, 4 * MB * MC * Fl, cudaMemcpyDeviceToDevice, s), "copy");
            return CSD_OK;
        case 6:
            CSD_CU(cudaMemcpyAsync(out, blk->aidx, 4 * B * Hl * C * blk->a_kmax, cudaMemcpyDeviceToDevice, s), "copy");
            if (counts_out)
                CSD_CU(cudaMemcpyAsync(counts_out, blk->acnt, 4 * B * Hl * C, cudaMemcpyDeviceToDevice, s), "copy");
            return CSD_OK;
        case 7: {
            const int64_t mk = c.mlp_k > 0 ? c.mlp_k : Fl;
            CSD_CU(cudaMemcpyAsync(out, blk->midx, 4 * MB * MC * mk, cudaMemcpyDeviceToDevice, s), "copy");
            if (counts_out)
                CSD_CU(cudaMemcpyAsync(counts_out, blk->mcnt, 4 * MB * MC, cudaMemcpyDeviceToDevice, s), "copy");
            return CSD_OK;
        }
    }
    (void)E;
    return set_error(CSD_ERR_VALUE, "unknown cache view %d", which);
}

}  // extern "C"
