// kernels.h — internal launcher declarations (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace csd {
namespace dev {

// Device-side error flags (checked by csd_ctx_sync).  Kernels that validate
// data set a bit and keep going; the host maps the first bit to a status.
enum : uint32_t {
    kFlagIndexRange = 1u << 0,
    kFlagIndexDup = 1u << 1,
    kFlagNonFinite = 1u << 2,
    kFlagCountRange = 1u << 3,
};

// ---- check mode (check_kernels.cu) ----------------------------------------
cudaError_t check_attention_logits(const float* q, const float* k, int layout, int64_t batch,
                                   int64_t heads, int64_t n, int64_t e, int64_t chunk,
                                   const int32_t* idx, const int32_t* counts, int64_t k_max,
                                   float* logits, cudaStream_t s);
cudaError_t check_softmax(float* buf, int64_t rows, int64_t rows_per_batch, int64_t stride,
                          const int32_t* counts, int64_t full, float* row_max, float* exp_sum,
                          uint32_t* flags, cudaStream_t s);
cudaError_t check_attention_pv(const float* probs, const float* v, int layout, int64_t batch,
                               int64_t heads, int64_t n, int64_t e, int64_t chunk,
                               const int32_t* idx, const int32_t* counts, int64_t k_max,
                               const float* base, float scale, float* out, cudaStream_t s);
cudaError_t check_colsum(const float* logits, const float* m, const float* l, int64_t bh_count,
                         int64_t n, int64_t chunk, float* out, cudaStream_t s);
cudaError_t check_project(const float* x, const float* w, int64_t batch, int64_t n, int64_t d,
                          int64_t dout, float* out, cudaStream_t s);
cudaError_t check_add(const float* a, const float* b, int64_t numel, float* out, cudaStream_t s);
cudaError_t check_dense_mlp(const float* x, const float* w1, const float* b1, const float* w2,
                            const float* b2, int64_t batch, int64_t n, int64_t d, int64_t f,
                            float* act_ref, float* out, cudaStream_t s);
cudaError_t check_mlp_preact(const float* x, const float* w1, const float* b1, int64_t rows,
                             int64_t d, int64_t f, float* pre, cudaStream_t s);
cudaError_t check_tile_means(const float* x, const float* w1, int64_t batch, int64_t n, int64_t d,
                             int64_t f, int64_t chunk, float* means_ws, float* out,
                             cudaStream_t s);
cudaError_t check_absdiff(const float* a, const float* b, int64_t numel, float* out,
                          cudaStream_t s);
cudaError_t check_sparse_delta_mlp(const float* x, const float* w1, const float* b1,
                                   const float* w2, const int32_t* idx, const int32_t* counts,
                                   int64_t k_max, int64_t chunk, int64_t batch, int64_t n,
                                   int64_t d, int64_t f, float* act_ref, float* out_cache,
                                   float* ws, cudaStream_t s);

// ---- shared (both modes) ---------------------------------------------------
// topk.cu
cudaError_t topk_rows(const float* scores, int64_t rows, int64_t m, int64_t k, int32_t* idx,
                      int32_t* counts, cudaStream_t s, bool sorted = true);
int64_t topk_max_k();
bool topk_cluster_eligible(int64_t rows, int64_t m);
cudaError_t topk_rows_fused_absdiff(const float* partial, int ks, const float* cached, int64_t rows,
                                    int64_t m, int64_t k, int32_t* idx, int32_t* counts,
                                    cudaStream_t s);
cudaError_t topk_rows_global(const float* scores, int64_t rows, int64_t m, int64_t k,
                             int32_t* idx, int32_t* counts, uint64_t* ws, cudaStream_t s);
cudaError_t validate_index_set(const int32_t* idx, const int32_t* counts, int64_t rows,
                               int64_t k_max, int64_t domain, uint32_t* flags, cudaStream_t s);
// shard.cu (F-sharded exact selection)
cudaError_t shard_candidates(const int32_t* ids, const float* scores, int64_t rows, int64_t m,
                             int64_t k_loc, int64_t k_out, int64_t id_offset, float* cand_scores,
                             int32_t* cand_ids, cudaStream_t s);
cudaError_t shard_merge(const float* all_scores, const int32_t* all_ids, int64_t g, int64_t rows,
                        int64_t k, int64_t f0, int64_t f_local, float* ws_scores, int32_t* ws_ids,
                        int32_t* ws_pos, int32_t* ws_cnt, int32_t* idx, int64_t ld_idx,
                        int32_t* counts, cudaStream_t s);
// voxel.cu
cudaError_t voxel_reorder(const void* src, void* dst, int64_t batch, int64_t t, int64_t h,
                          int64_t w, int64_t vt, int64_t vh, int64_t vw, int64_t row_bytes,
                          int inverse, cudaStream_t s);

// ---- production (prod_kernels.cu / attn_tc.cu) -----------------------------
struct AttnTcArgs {
    const void* q;  // bf16
    const void* k;
    const void* v;
    const int32_t* idx;     // nullable = dense (all keys, contiguous TMA tiles)
    const int32_t* counts;  // per (b,h,chunk)
    int64_t k_max;
    const void* base;  // bf16, nullable
    float scale;       // out = base + scale * O / l   (or O / l without base)
    void* out;         // bf16
    float* row_max;    // nullable [B,H,N] (natural-log units, like softmax_rows)
    float* exp_sum;    // nullable
    const float* prev_m;  // nullable: colsum stats (fresh if null and colsum requested)
    const float* prev_l;
    float* colsum;     // nullable [B,H,N/c,N]
    int layout;
    int64_t batch, heads, n, e, chunk;
    // colsum chunk when the work items use a different row count (chunk = item rows; the
    // column sums are per cs_chunk rows, accumulated atomically into a zeroed colsum);
    // 0 = the item rows
    int64_t cs_chunk;
    // sparse: work position -> item, longest first (lpt_order), or null (identity order)
    const int32_t* order;
};
// Longest-processing-time order of the (b, h, chunk) items of a ragged index set: items
// sorted stably by descending key-block count (counting sort, one CTA) into order[0, items),
// order[items] = 1 when that is the identity; persistent CTAs then take positions b,
// b + grid, ... (attn_pp.cu).
cudaError_t lpt_order(const int32_t* counts, int64_t items, int64_t block_keys, int32_t* order,
                      cudaStream_t s);
// Returns cudaErrorNotSupported for shapes outside the envelope.
cudaError_t attn_tc(const AttnTcArgs& a, cudaStream_t s);
bool attn_tc_supported(int64_t e, int64_t chunk);
// attn_pp.cu: ping-pong-tile kernel for items of 129..256 rows without column sums
// (CSD_ATTN_KERNEL=tc forces k_attn_tc); attn_tc() dispatches to it.
bool attn_pp_supported(const AttnTcArgs& a);
// attn_sd.cu: dense passes (dense attention, stats, stale-stat column sums) with a
// double-buffered S and tensor-core column sums; attn_tc() dispatches to it first.
bool attn_sd_supported(const AttnTcArgs& a);
cudaError_t attn_sd(const AttnTcArgs& a, cudaStream_t s);
cudaError_t attn_pp(const AttnTcArgs& a, cudaStream_t s);
// attn_cp.cu: sparse delta attention on CTA pairs (chunk 192 / 256, E 128, with base);
// attn_tc() dispatches to it before the ping-pong kernel (CSD_ATTN_CP=0 turns it off).
bool attn_cp_supported(const AttnTcArgs& a);
// attn_px.cu: the ping-pong kernel with P staged in shared memory (SS-form P V, the S buffer
// released as soon as it is in registers); opt-in (CSD_ATTN_PX=1) while measured.
bool attn_px_supported(const AttnTcArgs& a);
cudaError_t attn_px(const AttnTcArgs& a, cudaStream_t s);
cudaError_t attn_cp(const AttnTcArgs& a, cudaStream_t s);

// gemm_tc.cu: persistent tcgen05 GEMMs with fused epilogues (projections, dense MLP).
// gemm_tc_enabled() is false when CSD_GEMM=cublas (A/B comparison against the library).
bool gemm_tc_enabled();
bool gemm_tc_proj_supported(int64_t rows, int64_t k, int64_t n);
// out_i[rows, n] = x[rows, k] @ w_i[k, n] for nw weights (one launch); with resid (nw = 1):
// out = resid + x @ w
cudaError_t gemm_tc_proj(const void* x, const void* const w[3], void* const out[3], int nw,
                         int64_t rows, int64_t k, int64_t n, const void* resid, cudaStream_t s);
cudaError_t gemm_tc_proj_blocked(const void* a_blocks, const void* w, void* out, int64_t rows,
                                 int64_t k, int64_t n, const void* resid, int64_t a_bk,
                                 int64_t a_brows, cudaStream_t s);
bool gemm_tc_mlp_supported(int64_t d, int64_t f, int64_t chunk);
cudaError_t gemm_tc_mlp_up(const void* x, const void* w1, const float* b1, int64_t chunks,
                           int64_t chunk, int64_t d, int64_t f, void* cm, cudaStream_t s);
cudaError_t gemm_tc_mlp_down(const void* cm, const void* w2, const float* b2, int64_t chunks,
                             int64_t chunk, int64_t d, int64_t f, float* mcache,
                             const void* x_mid, void* x_out, cudaStream_t s);

cudaError_t prod_cast_f32_bf16(const float* in, void* out, int64_t n, cudaStream_t s);
cudaError_t prod_cast_bf16_f32(const void* in, float* out, int64_t n, cudaStream_t s);

// prod MLP (prod_kernels.cu)
// means_tc.cu: tcgen05 tile means (T, or |T - cached| when cached != null)
bool means_tc_supported(int64_t d, int64_t f);
size_t prod_means_ws_bytes(int64_t batch, int64_t n, int64_t d, int64_t f, int64_t chunk);
// With partials_out the split-K partials are left in ws (not reduced into out) and
// described there, for a consumer that fuses the reduction.
struct MeansPartials {
    const float* partial;
    int ks;
};
cudaError_t prod_tile_means_tc(const void* x, const void* w1, int64_t batch, int64_t n,
                               int64_t d, int64_t f, int64_t chunk, const float* cached,
                               float* out, void* ws, cudaStream_t s,
                               MeansPartials* partials_out = nullptr);
// dense-step MLP epilogue: act = gelu(pre + b1) row-major + chunk-major cache copy
cudaError_t prod_bias_gelu_cm(const void* pre, const float* b1, int64_t batch, int64_t n,
                              int64_t f, int64_t chunk, void* act, void* cm, cudaStream_t s);
// out += b2 (rows); if x_out: x_out = bf16(x_mid + out)
cudaError_t prod_bias_add_rows(float* out, const float* b2, int64_t rows, int64_t d,
                               const void* x_mid, void* x_out, cudaStream_t s);
// residual adds for the block runner: out_bf16 = a_bf16 + b_f32
cudaError_t prod_add_bf16_f32(const void* a, const float* b, int64_t numel, void* out,
                              cudaStream_t s);// mlp_tc.cu: delta_ws >= B*C*chunk*round_up(k_max,128) bf16
bool mlp_tc_supported(int64_t d, int64_t chunk);
// delta-workspace columns (k_pad) the tcgen05 sparse-delta MLP uses for k_max / nz chunks
int64_t prod_smlp_delta_cols(int64_t k_max, int64_t nz, int64_t chunk);
cudaError_t prod_sparse_delta_mlp_tc(const void* x, const void* w1, const float* b1,
                                     const void* w2, const int32_t* idx, const int32_t* counts,
                                     int64_t k_max, int64_t chunk, int64_t batch, int64_t n,
                                     int64_t d, int64_t f, void* act_cm, float* out_cache,
                                     void* delta_ws, cudaStream_t s,
                                     const void* x_mid = nullptr, void* x_out = nullptr);
cudaError_t prod_act_cm_to_ref(const void* act_cm, int64_t batch, int64_t n, int64_t f,
                               int64_t chunk, float* out, cudaStream_t s);
cudaError_t prod_absdiff(const float* a, const float* b, int64_t numel, float* out,
                         cudaStream_t s);

}  // namespace dev
}  // namespace csd
