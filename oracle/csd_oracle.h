/*
 * csd_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's column-sparse-delta hot path
 * (/root/reference/proj/src/{tensor,voxel,sparse_index,attention,mlp,model}.cpp),
 * used as the parity checker for the CUDA product path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; the
 * product library (paper_2506_03275_b200/libcsd_b200.so) never links or calls it.
 *
 * Arithmetic contract (what makes bit-exact comparison possible):
 *   - every float op is a separate IEEE binary32 op in the reference's order
 *     (compiled with -ffp-contract=off, matching the reference's x86-64
 *     baseline build which has no FMA: SURVEY.md §8a row a16);
 *   - exp / tanh are restatements of glibc 2.39 expf / tanhf (the functions
 *     std::exp / std::tanh resolve to in the reference build), pinned
 *     against the host libm in tests/test_oracle.py.
 *
 * Layouts are the reference's row-major layouts ([B,H,N,E], [B,N,D], ...).
 * Functions return 0 on success or a negative CSDO_E* code (mirrors the
 * reference exception classes in include/csd/error.hpp:8-46).
 */
#ifndef CSD_ORACLE_H
#define CSD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    CSDO_OK = 0,
    CSDO_ESHAPE = -1,  /* ShapeError  */
    CSDO_EINDEX = -2,  /* IndexError  */
    CSDO_ENUMERIC = -3,/* NumericError */
    CSDO_ESTATE = -4,  /* StateError  */
    CSDO_EVALUE = -5,  /* ValueError  */
    CSDO_ECONFIG = -6, /* ConfigError */
};

/* glibc-2.39-compatible scalar transcendentals. */
float csdo_expf(float x);
float csdo_tanhf(float x);
float csdo_gelu(float x);

/* voxel.cpp:18-42 (permutation), :44-73 (gather), :75-102 (scatter) */
int csdo_voxel_permutation(int64_t t, int64_t h, int64_t w, int64_t vt, int64_t vh, int64_t vw,
                           int64_t* perm_out);
int csdo_voxel_order(const float* x, int64_t batch, int64_t t, int64_t h, int64_t w, int64_t d,
                     int64_t vt, int64_t vh, int64_t vw, float* out);
int csdo_reverse_voxel_order(const float* x, int64_t batch, int64_t t, int64_t h, int64_t w,
                             int64_t d, int64_t vt, int64_t vh, int64_t vw, float* out);

/* sparse_index.cpp:64-96: per-row top-k, descending score, lower index on ties. */
int csdo_select_top_k(const float* scores, int64_t rows, int64_t m, int64_t k, int32_t* idx_out);
/* sparse_index.cpp:27-62 */
int csdo_validate_index_set(const int32_t* idx, const int32_t* counts, int64_t rows, int64_t k_max,
                            int64_t domain);

/* tensor.cpp:66-98 (gemm), :100-139 (softmax_rows) */
void csdo_gemm(const float* a, const float* b, int64_t m, int64_t kk, int64_t n, int transpose_b,
               float* out);
int csdo_softmax_rows(const float* logits, int64_t rows, int64_t len, float* probs, float* row_max,
                      float* exp_sum);

/* attention.cpp:59-74 */
int csdo_dense_attention(const float* q, const float* k, const float* v, int64_t batch,
                         int64_t heads, int64_t n, int64_t e, float* out);
/* attention.cpp:76-145; prev_m/prev_l may be NULL (fresh stats). */
int csdo_column_sum_attention(const float* q, const float* k, const float* v, const float* prev_m,
                              const float* prev_l, int64_t batch, int64_t heads, int64_t n,
                              int64_t e, int64_t chunk, float* out, float* row_max,
                              float* exp_sum, float* column_sums);
/* attention.cpp:147-194 */
int csdo_sparse_delta_attention(const float* q, const float* k, const float* v,
                                const int32_t* idx, const int32_t* counts, int64_t k_max,
                                int64_t chunk, const float* base, float scale, int64_t batch,
                                int64_t heads, int64_t n, int64_t e, float* out);

/* mlp.cpp:49-81; pre/act may be NULL. */
int csdo_dense_mlp(const float* x, const float* w1, const float* b1, const float* w2,
                   const float* b2, int64_t batch, int64_t n, int64_t d, int64_t f, float* out,
                   float* pre, float* act);
/* mlp.cpp:83-96 */
int csdo_mlp_tile_means(const float* x, const float* w1, int64_t batch, int64_t n, int64_t d,
                        int64_t f, int64_t chunk, float* out);
/* mlp.cpp:98-118 */
int csdo_mlp_change_indices(const float* x, const float* w1, const float* tile_means,
                            int64_t batch, int64_t n, int64_t d, int64_t f, int64_t k,
                            int64_t chunk, int32_t* idx_out);
/* mlp.cpp:120-182: act_cache [B,N,F] and out_cache [B,N,D] updated in place. */
int csdo_sparse_delta_mlp(const float* x, const float* w1, const float* b1, const float* w2,
                          const int32_t* idx, const int32_t* counts, int64_t k_max,
                          int64_t chunk, int64_t batch, int64_t n, int64_t d, int64_t f,
                          float* act_cache, float* out_cache);

/* model.cpp:107-120 (x[B,N,D] @ w[D,Dout]), :122-165 (head split / merge) */
void csdo_project(const float* x, const float* w, int64_t batch, int64_t n, int64_t d,
                  int64_t dout, float* out);
void csdo_split_heads(const float* x, int64_t batch, int64_t n, int64_t heads, int64_t e,
                      float* out);
void csdo_merge_heads(const float* x, int64_t batch, int64_t heads, int64_t n, int64_t e,
                      float* out);

/* rng.hpp:12-44 seeded Gaussian stream (tests/test_util.hpp:50-55). */
void csdo_gaussian(uint64_t seed, int64_t n, float stddev, float* out);
/* Mismatch count vs host libm (which: 0 expf, 1 tanhf) over a bit-pattern range. */
int64_t csdo_libm_mismatches(uint32_t start, uint32_t stop, uint32_t step, int which);

#ifdef __cplusplus
}
#endif

#endif
