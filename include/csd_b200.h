/*
 * csd_b200.h — C ABI of the B200-native Chipmunk column-sparse-delta path.
 *
 * This is the drop-in boundary: plain pointers, sizes and status codes, no
 * C++/torch types.  Every entry point replaces one routine of the reference's
 * C++ operator API (namespace csd, /root/reference/proj/include/csd/*.hpp);
 * the replaced declaration is cited on each function.  The host-side C++
 * mirror of that API (include/csd/*.hpp, libcsd_host.so) and the Python
 * binding (paper_2506_03275_b200/_capi.py) are both thin layers over this.
 *
 * Conventions
 *  - Tensor pointers are DEVICE pointers (cudaMalloc / torch CUDA storage),
 *    row-major, in the reference's layouts unless a `layout` argument says
 *    otherwise.  `stream` is a cudaStream_t passed as void* (NULL = legacy
 *    default stream).  Calls are stream-ordered and asynchronous except
 *    where noted; validation that needs device data (index uniqueness,
 *    non-finite logits) happens in-kernel and is reported by csd_ctx_sync().
 *  - mode CSD_MODE_CHECK: fp32 storage, bit-exact reproduction of the
 *    reference arithmetic (sequential fp32 accumulation, no FMA contraction,
 *    glibc-2.39-compatible expf/tanhf).  Any shape the reference accepts.
 *  - mode CSD_MODE_PROD: bf16 activations/weights, fp32 accumulation on
 *    tcgen05 tensor cores (TMEM accumulators, TMA-gathered operand tiles).
 *    Shapes outside a kernel's envelope return CSD_ERR_UNSUPPORTED — there is
 *    no CPU or eager fallback.
 *  - Index sets follow SparseIndexSet (sparse_index.hpp:15-40): indices
 *    int32 [rows * k_max], counts int32 [rows], rows = B*H*C (H = 1 for MLP).
 *  - Errors: a csd_status; csd_last_error() returns a thread-local message
 *    naming the offending value, mirroring the reference exception text.
 */
#ifndef CSD_B200_H
#define CSD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSD_ABI_VERSION 1

/* Status codes <-> reference exception classes (error.hpp:8-46). */
typedef enum {
    CSD_OK = 0,
    CSD_ERR_SHAPE = 1,       /* ShapeError   */
    CSD_ERR_INDEX = 2,       /* IndexError   */
    CSD_ERR_NUMERIC = 3,     /* NumericError */
    CSD_ERR_STATE = 4,       /* StateError   */
    CSD_ERR_VALUE = 5,       /* ValueError   */
    CSD_ERR_CONFIG = 6,      /* ConfigError  */
    CSD_ERR_CUDA = 7,        /* CUDA runtime / launch failure */
    CSD_ERR_UNSUPPORTED = 8  /* shape outside the production kernel envelope */
} csd_status;

typedef enum { CSD_MODE_CHECK = 0, CSD_MODE_PROD = 1 } csd_mode;

/* Attention tensor layouts: reference [B,H,N,E] or token-major [B,N,H,E]
 * (what a fused x@Wq projection produces; avoids split/merge_heads copies,
 * model.cpp:122-165). */
typedef enum { CSD_LAYOUT_BHNE = 0, CSD_LAYOUT_BNHE = 1 } csd_layout;

typedef struct csd_ctx csd_ctx;

int csd_abi_version(void);
const char* csd_last_error(void);
const char* csd_status_name(csd_status s);

/* Context: device binding, scratch workspace, side stream, error flag. */
csd_status csd_ctx_create(int device, csd_ctx** out);
csd_status csd_ctx_destroy(csd_ctx* ctx);
/* Synchronises `stream` and surfaces in-kernel validation failures
 * (duplicate / out-of-range ids, non-finite logits) as the matching status. */
csd_status csd_ctx_sync(csd_ctx* ctx, void* stream);
/* Device memory helpers for hosts that do not link the CUDA runtime themselves (the C++
 * csd:: mirror).  Synchronous copies on the legacy default stream. */
csd_status csd_device_alloc(size_t bytes, void** out);
csd_status csd_device_free(void* ptr);
csd_status csd_copy_to_device(void* dst, const void* src, size_t bytes);
csd_status csd_copy_to_host(void* dst, const void* src, size_t bytes);
/* Element conversion between fp32 and bf16 device buffers (round to nearest even):
 * to_bf16 != 0: src fp32 -> dst bf16, else src bf16 -> dst fp32. */
csd_status csd_cast(csd_ctx* ctx, const void* src, void* dst, int64_t n, int to_bf16, void* stream);
/* PROD-mode index-set validation on every sparse call (default on; the block
 * runner disables it for its own top-k sets, which are valid by construction). */
csd_status csd_ctx_set_validation(csd_ctx* ctx, int enabled);
/* select_top_k output order (default 1: descending score, lower index first on ties,
 * sparse_index.cpp:86-90).  0: the same exact index SET, strictly-greater entries then the
 * lowest-index ties, each in index order (what the PROD block path uses: its consumers are
 * order-invariant; lets few long rows run as a cluster of CTAs per row). */
csd_status csd_ctx_set_sorted_topk(csd_ctx* ctx, int sorted);
/* Longest-first (LPT) order of the (b, h, chunk) work items of PROD sparse attention over a
 * ragged index set (default on; one small ordering kernel per call).  Results do not depend
 * on it. */
csd_status csd_ctx_set_lpt(csd_ctx* ctx, int enabled);
/* Number of kernels this context launched since creation (instrumentation). */
int64_t csd_ctx_launch_count(const csd_ctx* ctx);

/* ---------------------------------------------------------------- voxel --
 * voxel.hpp:30-36.  The permutation is computed on the host; the device
 * reorder derives it arithmetically per row (no index array in HBM).      */
/* voxel_permutation (voxel.cpp:18-42): perm_out[N] on the HOST. */
csd_status csd_voxel_permutation(int64_t t, int64_t h, int64_t w, int64_t vt, int64_t vh,
                                 int64_t vw, int64_t* perm_out);
/* voxel_order (inverse=0, voxel.cpp:44-73) / reverse_voxel_order (inverse=1,
 * voxel.cpp:75-102) for rows of `row_bytes` bytes (any dtype; bit-exact). */
csd_status csd_voxel_reorder(csd_ctx* ctx, const void* src, void* dst, int64_t batch, int64_t t,
                             int64_t h, int64_t w, int64_t vt, int64_t vh, int64_t vw,
                             int64_t row_bytes, int inverse, void* stream);

/* ---------------------------------------------------------------- top-k --
 * select_top_k (sparse_index.hpp:45, sparse_index.cpp:64-96): per row of m
 * fp32 scores keep the k largest, lower index first on ties, stored in
 * descending-score order; counts[row] = k.  Exact in both modes. */
csd_status csd_select_top_k(csd_ctx* ctx, const float* scores, int64_t rows, int64_t m, int64_t k,
                            int32_t* idx, int32_t* counts, void* stream);
/* SparseIndexSet::validate (sparse_index.cpp:27-62), on device. */
csd_status csd_validate_index_set(csd_ctx* ctx, const int32_t* idx, const int32_t* counts,
                                  int64_t rows, int64_t k_max, int64_t domain, void* stream);

/* ------------------------------------------------------------ attention --
 * dtype: CHECK -> float tensors; PROD -> bf16 q/k/v/out/base, fp32 stats. */
/* dense_attention (attention.hpp:30-33, attention.cpp:59-74). */
csd_status csd_dense_attention(csd_ctx* ctx, csd_mode mode, csd_layout layout, const void* q,
                               const void* k, const void* v, int64_t batch, int64_t heads,
                               int64_t n, int64_t e, void* out, void* stream);
/* column_sum_attention (attention.hpp:35-41, attention.cpp:76-145).
 * prev_m/prev_l [B,H,N] may be NULL (fresh stats).  Outputs: out, row_max,
 * exp_sum [B,H,N] (fp32) and column_sums [B,H,N/chunk,N] (fp32). */
csd_status csd_column_sum_attention(csd_ctx* ctx, csd_mode mode, csd_layout layout,
                                    const void* q, const void* k, const void* v,
                                    const float* prev_m, const float* prev_l, int64_t batch,
                                    int64_t heads, int64_t n, int64_t e, int64_t chunk, void* out,
                                    float* row_max, float* exp_sum, float* column_sums,
                                    void* stream);
/* sparse_delta_attention (attention.hpp:43-47, attention.cpp:147-194):
 * out = base + scale * softmax(q_c K_S^T / sqrt(E)) V_S per chunk; count 0
 * chunks copy base bit-exactly.  base may alias out. */
csd_status csd_sparse_delta_attention(csd_ctx* ctx, csd_mode mode, csd_layout layout,
                                      const void* q, const void* k, const void* v,
                                      const int32_t* idx, const int32_t* counts, int64_t k_max,
                                      int64_t chunk, const void* base, float scale,
                                      int64_t batch, int64_t heads, int64_t n, int64_t e,
                                      void* out, void* stream);

/* ------------------------------------------------------------------ MLP --
 * Weights: w1, w2 [F,D] (neuron-major, mlp.hpp:12-21), b1 [F], b2 [D].
 * CHECK: all fp32.  PROD: x/w1/w2 bf16, biases fp32, act cache bf16 in the
 * chunk-major layout [B, N/c, F, c], output cache fp32 [B,N,D]. */
/* dense_mlp (mlp.hpp:44, mlp.cpp:49-81).  act_out (nullable) receives the
 * activations in the mode's act-cache layout. */
csd_status csd_dense_mlp(csd_ctx* ctx, csd_mode mode, const void* x, const void* w1,
                         const float* b1, const void* w2, const float* b2, int64_t batch,
                         int64_t n, int64_t d, int64_t f, int64_t chunk, float* out,
                         void* act_out, void* stream);
/* MlpDenseResult::preact (mlp.cpp:55-59): pre = x W1^T + b1, [B,N,F] fp32.  CHECK only. */
csd_status csd_mlp_preact(csd_ctx* ctx, csd_mode mode, const void* x, const void* w1,
                          const float* b1, int64_t batch, int64_t n, int64_t d, int64_t f,
                          float* pre_out, void* stream);
/* mlp_tile_means (mlp.hpp:47, mlp.cpp:83-96): out [B, N/c, F] fp32. */
csd_status csd_mlp_tile_means(csd_ctx* ctx, csd_mode mode, const void* x, const void* w1,
                              int64_t batch, int64_t n, int64_t d, int64_t f, int64_t chunk,
                              float* out, void* stream);
/* mlp_change_indices (mlp.hpp:51-53, mlp.cpp:98-118). */
csd_status csd_mlp_change_indices(csd_ctx* ctx, csd_mode mode, const void* x, const void* w1,
                                  const float* tile_means, int64_t batch, int64_t n, int64_t d,
                                  int64_t f, int64_t k, int64_t chunk, int32_t* idx,
                                  int32_t* counts, void* stream);
/* sparse_delta_mlp (mlp.hpp:55-60, mlp.cpp:120-182): act_cache and
 * out_cache updated in place (O = O_cache + delta); out (nullable) gets a
 * copy of the new output in the mode's activation dtype. */
csd_status csd_sparse_delta_mlp(csd_ctx* ctx, csd_mode mode, const void* x, const void* w1,
                                const float* b1, const void* w2, const int32_t* idx,
                                const int32_t* counts, int64_t k_max, int64_t chunk,
                                int64_t batch, int64_t n, int64_t d, int64_t f, void* act_cache,
                                float* out_cache, void* stream);
/* Convert a mode's act cache to the reference layout [B,N,F] fp32 (for the
 * host mirror's MlpCache::activations view, test_mlp.cpp:234). */
csd_status csd_mlp_act_cache_to_ref(csd_ctx* ctx, csd_mode mode, const void* act_cache,
                                    int64_t batch, int64_t n, int64_t f, int64_t chunk,
                                    float* out, void* stream);

/* --------------------------------------------------------------- dense ops --
 * project (model.cpp:107-120): out[B,N,Dout] = x[B,N,D] @ w[D,Dout]; and the
 * residual add (model.cpp:47-57).  CHECK only (PROD projections live inside
 * the block runner). */
csd_status csd_project(csd_ctx* ctx, csd_mode mode, const void* x, const void* w, int64_t batch,
                       int64_t n, int64_t d, int64_t dout, void* out, void* stream);
csd_status csd_add(csd_ctx* ctx, csd_mode mode, const void* a, const void* b, int64_t numel,
                   void* out, void* stream);

/* ----------------------------------------------------------- generation --
 * The multi-step schedule driver's pieces.
 *
 * csd_resolve_schedule replaces csd::resolve_schedule (schedule.cpp:44-87, with the
 * StepSchedule::validate invariants :21-41): modes[total_steps] receives csd_step_mode
 * values — a dense refresh at step 0 and every (dense_interval + 1) boundary, sparse in
 * between; with the step cache, steps of the centred `window` that are off the `stride`
 * grid are skipped (step 0 never is).  Host-only; CSD_ERR_CONFIG on the reference's
 * ConfigError cases. */
typedef enum { CSD_STEP_DENSE = 0, CSD_STEP_SPARSE = 1, CSD_STEP_SKIPPED = 2 } csd_step_mode;
csd_status csd_resolve_schedule(int64_t total_steps, int64_t dense_interval, int use_step_cache,
                                int64_t window, int64_t stride, int32_t* modes);
/* latent[i] += a * y[i] (harness.cpp:24-30, the per-step update at :200).  The latent is
 * an fp32 master in both modes; y is the model output (fp32 CHECK, bf16 PROD).  PROD also
 * writes bf16(latent) into latent_bf16 when non-null (the next step's block input). */
csd_status csd_latent_axpy(csd_ctx* ctx, csd_mode mode, float* latent, float a, const void* y,
                           int64_t numel, void* latent_bf16, void* stream);
/* R^2 of (truth - origin) vs (approx - origin), fp32 inputs, double accumulation
 * (metrics.cpp:5-30 over the harness.cpp:32-38 deltas; origin may be NULL).  Deterministic
 * device reduction; synchronises `stream` and writes *r2 on the host.  CSD_ERR_NUMERIC when
 * the true delta has zero variance (the reference's NumericError). */
csd_status csd_r_squared(csd_ctx* ctx, const float* truth, const float* approx,
                         const float* origin, int64_t numel, double* r2, void* stream);
/* index_set_to_masks (bitmask.cpp:55-85): one bitpacked mask per
 * (b, h, chunk) row of an index set -- masks[rows][ceil(n_bits / 8)] bytes, bit i of byte j
 * = element 8 j + i (bitmask.hpp:13-17), trailing pad bits zero.  Validates like the
 * reference (ids in [0, n_bits) and unique -> CSD_ERR_INDEX; counts in [0, k_max] ->
 * CSD_ERR_VALUE); synchronises `stream`. */
csd_status csd_index_set_to_masks(csd_ctx* ctx, const int32_t* idx, const int32_t* counts,
                                  int64_t rows, int64_t k_max, int64_t n_bits, uint8_t* masks,
                                  void* stream);

/* ---------------------------------------------------------------- block --
 * One DiT block (model.cpp:178-216: x += attn(x Wq, x Wk, x Wv) Wo;
 * x += mlp(x)) with device-resident weights and per-layer caches
 * (AttentionCache / MlpCache, attention.hpp:13-19, mlp.hpp:29-36).
 * Head / hidden sharding: a block may own heads [head0, head0+heads_local)
 * and neurons [f0, f0+f_local) (csd_block_config); sharded execution is
 * driven through the csd_block_*_partial calls below. */
typedef struct {
    int64_t batch, seq, dim, heads, head_dim, hidden, chunk;
    int64_t attn_k, mlp_k;   /* per-chunk keys / neurons recomputed */
    int64_t head0, heads_local, f0, f_local;  /* shard (0, heads, 0, hidden) = whole block */
    /* token-sharded execution: this rank's output projection and MLP run on token rows
     * [t0, t0 + t_local) of the B*N rows (chunk-aligned); 0, 0 = not token-sharded */
    int64_t t0, t_local;
} csd_block_config;

typedef struct csd_block csd_block;

/* Weights are HOST fp32 in reference layout (wq..wo [D,D], w1/w2 [F,D],
 * b1 [F], b2 [D]); the block keeps device copies in the mode's dtype. */
csd_status csd_block_create(csd_ctx* ctx, csd_mode mode, const csd_block_config* cfg,
                            const float* wq, const float* wk, const float* wv, const float* wo,
                            const float* w1, const float* b1, const float* w2, const float* b2,
                            csd_block** out);
csd_status csd_block_destroy(csd_block* blk);
/* Forget every cache (a fresh ModelState, model.cpp:101-105): the next step must be dense
 * and computes its column sums with fresh softmax stats. */
csd_status csd_block_reset(csd_block* blk);
/* model_forward_step for one layer: x_out = block(x_in).  x in the mode's
 * activation dtype, [B,N,D] device.  dense = 1 refreshes the caches; dense = 2 is
 * model_forward_dense (model.cpp:167-176): exact attention + dense MLP, the caches left
 * untouched (the dense baseline trajectory; scratch allocated on first use, so run it once
 * outside a graph capture first).
 * static_idx/static_counts (nullable, device) replace the attention top-k
 * on dense steps (attention.hpp:50-52): int32 [B, heads_local, N/chunk, static_k_max]
 * and [B, heads_local, N/chunk], static_k_max == cfg.attn_k.  The pattern is validated
 * before anything runs (CSD_ERR_SHAPE / CSD_ERR_INDEX / CSD_ERR_VALUE leave every cache
 * untouched; synchronous unless the stream is capturing, then reported by csd_ctx_sync).
 * A sparse step before any dense step returns CSD_ERR_STATE. */
csd_status csd_block_step(csd_block* blk, const void* x_in, void* x_out, int dense,
                          const int32_t* static_idx, const int32_t* static_counts,
                          int64_t static_k_max, void* stream);
/* ---- Sharded execution (PROD): heads [head0, +heads_local) and neurons [f0, +f_local) per
 * rank; the caller provides the collectives (NCCL over NVLink).  One step on rank r of g:
 *   csd_block_attn_partial(x_in -> attn_partial)        ; all-reduce(sum) attn_partial
 *   csd_residual_add(x_in, attn_partial -> x_mid)
 *   dense : csd_block_mlp_dense_partial(x_mid -> mlp_partial)
 *   sparse: csd_block_mlp_candidates(x_mid -> cand_scores, cand_ids [rows, k])
 *           all-gather candidates in rank order -> [g, rows, k]
 *           csd_block_mlp_sparse_partial(x_mid, all_scores, all_ids, g -> mlp_partial)
 *   all-reduce(sum) mlp_partial ; csd_residual_add(x_mid, mlp_partial -> x_out)
 * rows = B * N / chunk; k = cfg.mlp_k.  The merged selection is exactly the single-GPU
 * per-chunk top-k (global id tie rule); each rank keeps its own neurons. */
csd_status csd_block_attn_partial(csd_block* blk, const void* x_in, int dense,
                                  float* attn_partial, void* stream);
csd_status csd_block_mlp_dense_partial(csd_block* blk, const void* x_mid, float* mlp_partial,
                                       void* stream);
csd_status csd_block_mlp_candidates(csd_block* blk, const void* x_mid, float* cand_scores,
                                    int32_t* cand_ids, void* stream);
csd_status csd_block_mlp_sparse_partial(csd_block* blk, const void* x_mid,
                                        const float* all_scores, const int32_t* all_ids,
                                        int64_t world, float* mlp_partial, void* stream);
/* ---- Token-sharded execution (PROD, csd_block_config.t_local > 0): attention
 * by heads, the output projection and the MLP by token rows; the caller's collectives move
 * bf16 only.  One step on rank r of g (equal heads per rank, equal chunk-aligned rows):
 *   csd_block_attn_heads(x_in [B*N, D] -> attn_local [B*N, heads_local*E])
 *   all-to-all: rows [t0_s, +t_local) of attn_local to rank s   -> attn_rows [g][t_local][Dl]
 *   csd_block_rows_step(x_in rows [t0, +t_local), attn_rows, g -> x_out rows)
 *   all-gather x_out rows in rank order                         -> x_out [B*N, D]
 * The MLP selection and caches are per chunk, so the rows step is exactly the single-GPU
 * step on those rows (weights wo / w1 / w2 replicated). */
csd_status csd_block_attn_heads(csd_block* blk, const void* x_in, int dense, void* attn_local,
                                void* stream);
csd_status csd_block_rows_step(csd_block* blk, const void* x_rows, const void* attn_rows,
                               int64_t world, int dense, void* x_out_rows, void* stream);
/* out_bf16 = bf16(x_bf16 + partial_f32) (PROD residual after an all-reduce). */
csd_status csd_residual_add(csd_ctx* ctx, const void* x, const float* partial, int64_t numel,
                            void* out, void* stream);
/* Cache arena (memory.cpp:33-58): a block's persistent caches -- attention residual, softmax
 * stats, index sets, MLP activations / outputs / tile means -- live in one device
 * allocation.  csd_block_cache_arena reports it; csd_block_bind_cache_arena re-points the
 * caches into caller storage of at least that size (same layout, contents not copied; the
 * block's own arena is freed), so a layer stack can keep two arenas on the device and stream
 * the rest to host memory (generation.Generation(offload=True)). */
csd_status csd_block_cache_arena(csd_block* blk, void** dev_ptr, size_t* bytes);
csd_status csd_block_bind_cache_arena(csd_block* blk, void* dev_ptr, size_t bytes);

/* Cache views (reference layouts, fp32, device): which = 0 attn residual
 * [B,H,N,E], 1 row_max, 2 exp_sum [B,H,N], 3 mlp act [B,N,F], 4 mlp out
 * [B,N,D], 5 tile means [B,C,F]; 6/7 attention / mlp index sets (int32). */
csd_status csd_block_cache(csd_block* blk, int which, void* out, int32_t* counts_out,
                           void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CSD_B200_H */
