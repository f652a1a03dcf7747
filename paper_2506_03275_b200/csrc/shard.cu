// shard.cu — exact global MLP selection under hidden-column (F) sharding.
//
// Each of g ranks owns neurons [f0, f0 + F_r).  mlp_change_indices (mlp.cpp:98-118) needs
// the global per-chunk top-k of |T - T_m| with the reference order (score desc, neuron id
// asc).  The global top-k is a subset of the union of the per-shard top-k lists, so:
//   candidates : local top-k, re-sorted by ascending global id, scores gathered alongside
//                (padded with score -1 / id INT_MAX to exactly k entries);
//   (host)     : all-gather the [rows, k] candidate lists in rank order;
//   merge      : per row, the g*k candidates are laid out rank-major = ascending global id,
//                so the ordinary top-k kernel's "lower position wins ties" IS the reference
//                tie rule; positions map back to ids and each rank keeps its own shard's
//                ids (descending-score order preserved; counts vary per rank and chunk).
#include <climits>

#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace csd {
namespace dev {

// per row: ids (unique, k of them) -> ascending order; out_ids += id_offset, scores gathered
__global__ void k_candidates(const int32_t* __restrict__ ids, const float* __restrict__ scores,
                             int64_t m, int64_t k_loc, int64_t k_out, int64_t id_offset,
                             float* __restrict__ cand_scores, int32_t* __restrict__ cand_ids) {
    extern __shared__ int32_t s_ids[];
    const int64_t row = blockIdx.x;
    const int32_t* src = ids + row * k_loc;
    for (int i = threadIdx.x; i < k_loc; i += blockDim.x) s_ids[i] = src[i];
    __syncthreads();
    for (int i = threadIdx.x; i < k_loc; i += blockDim.x) {
        const int32_t v = s_ids[i];
        int rank = 0;
        for (int q = 0; q < k_loc; ++q) rank += s_ids[q] < v;
        cand_ids[row * k_out + rank] = v + (int32_t)id_offset;
        cand_scores[row * k_out + rank] = scores[row * m + v];
    }
    for (int i = (int)k_loc + threadIdx.x; i < k_out; i += blockDim.x) {
        cand_ids[row * k_out + i] = INT_MAX;
        cand_scores[row * k_out + i] = -1.0f;  // |dT| >= 0: padding never wins
    }
}

// [g][rows][k] -> [rows][g*k]
__global__ void k_rank_major_rows(const float* __restrict__ s_in, const int32_t* __restrict__ i_in,
                                  int64_t g, int64_t rows, int64_t k, float* __restrict__ s_out,
                                  int32_t* __restrict__ i_out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= g * rows * k) return;
    const int64_t r = e / (rows * k), row = (e / k) % rows, j = e % k;
    s_out[row * g * k + r * k + j] = s_in[e];
    i_out[row * g * k + r * k + j] = i_in[e];
}

// keep this rank's ids from the merged (descending) list: one warp per row, ordered compaction
__global__ void k_keep_local(const int32_t* __restrict__ pos, const int32_t* __restrict__ gids,
                             int64_t rows, int64_t gk, int64_t k, int64_t f0, int64_t f_local,
                             int32_t* __restrict__ idx, int64_t ld_idx, int32_t* __restrict__ counts) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    int32_t n = 0;
    for (int64_t j0 = 0; j0 < k; j0 += 32) {
        const int64_t j = j0 + lane;
        int32_t gid = -1;
        if (j < k) gid = gids[row * gk + pos[row * k + j]];
        const bool mine = j < k && gid >= f0 && gid < f0 + f_local;
        const uint32_t b = __ballot_sync(0xffffffffu, mine);
        if (mine) idx[row * ld_idx + n + __popc(b & ((1u << lane) - 1u))] = gid - (int32_t)f0;
        n += __popc(b);
    }
    if (lane == 0) counts[row] = n;
}

cudaError_t shard_candidates(const int32_t* ids, const float* scores, int64_t rows, int64_t m,
                             int64_t k_loc, int64_t k_out, int64_t id_offset, float* cand_scores,
                             int32_t* cand_ids, cudaStream_t s) {
    k_candidates<<<(unsigned)rows, 256, sizeof(int32_t) * k_loc, s>>>(ids, scores, m, k_loc, k_out,
                                                                      id_offset, cand_scores, cand_ids);
    return cudaGetLastError();
}

cudaError_t shard_merge(const float* all_scores, const int32_t* all_ids, int64_t g, int64_t rows,
                        int64_t k, int64_t f0, int64_t f_local, float* ws_scores, int32_t* ws_ids,
                        int32_t* ws_pos, int32_t* ws_cnt, int32_t* idx, int64_t ld_idx,
                        int32_t* counts, cudaStream_t s) {
    const int64_t tot = g * rows * k;
    k_rank_major_rows<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(all_scores, all_ids, g, rows, k,
                                                                     ws_scores, ws_ids);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = topk_rows(ws_scores, rows, g * k, k, ws_pos, ws_cnt, s);
    if (e != cudaSuccess) return e;
    k_keep_local<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(ws_pos, ws_ids, rows, g * k, k, f0, f_local,
                                                            idx, ld_idx, counts);
    return cudaGetLastError();
}

}  // namespace dev
}  // namespace csd
