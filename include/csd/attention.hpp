// csd/attention.hpp — Chipmunk column-sparse attention (reference attention.hpp:13-52).
// Every function runs on the B200 through libcsd_b200.so (CSD_MODE_CHECK): the results are
// bit-identical to the reference CPU implementation.
#pragma once

#include <cstdint>

#include "csd/sparse_index.hpp"
#include "csd/tensor.hpp"

namespace csd {

struct AttentionCache {
    Tensor residual_output;  // [B, H, N, E]: dense output minus the recomputable sparse part
    SoftmaxStats stats;      // row constants of the last dense step
    SparseIndexSet indices;
    int64_t age = 0;
    bool initialized = false;
};

struct ColumnSumAttentionResult {
    Tensor output;       // [B, H, N, E]
    Tensor column_sums;  // [B, H, N/c, N]
    SoftmaxStats stats;  // fresh
};

Tensor dense_attention(const Tensor& q, const Tensor& k, const Tensor& v);
ColumnSumAttentionResult column_sum_attention(const Tensor& q, const Tensor& k, const Tensor& v,
                                              const SoftmaxStats* prev_stats, int64_t chunk);
Tensor sparse_delta_attention(const Tensor& q, const Tensor& k, const Tensor& v,
                              const SparseIndexSet& indices, const Tensor& base, float scale);
Tensor attention_step(const Tensor& q, const Tensor& k, const Tensor& v, AttentionCache& cache,
                      bool dense_step, int64_t top_k, int64_t chunk,
                      const SparseIndexSet* static_indices = nullptr);

}  // namespace csd
