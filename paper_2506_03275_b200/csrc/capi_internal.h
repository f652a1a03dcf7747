// capi_internal.h — host-side context shared by the C-ABI translation units.
#pragma once

#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <mutex>
#include <utility>
#include <vector>

#include "csd_b200.h"
#include "kernels.h"

namespace csd {

enum WsSlot {
    kWsTopk = 0,
    kWsLogits,
    kWsProbs,
    kWsStatsM,
    kWsStatsL,
    kWsMeans,
    kWsScores,
    kWsDelta,
    kWsPre,
    kWsAct,
    kWsIdx,
    kWsCounts,
    kWsR2,
    kWsOrder,
    kWsCount
};

struct Ctx {
    int device = 0;
    int sm_count = 0;
    uint32_t* flags = nullptr;  // device error bits (kFlag*)
    cublasHandle_t cublas = nullptr;
    std::vector<std::pair<void*, size_t>> bufs;
    std::vector<void*> retired;  // grown-out workspaces (graphs may still reference them)
    std::mutex mu;
    int64_t launches = 0;          // our kernels launched through this context
    int64_t library_launches = 0;  // cuBLAS GEMM calls
    bool validate_prod = true;     // PROD-mode async index validation
    // select_top_k output order: descending score (the reference contract, sparse_index.cpp:
    // 86-90).  The PROD block path clears it: its consumers (column-sparse attention,
    // sparse-delta MLP) are order-invariant, so the same exact index SET in index order
    // skips the per-row sort.
    bool sorted_topk = true;
    // sparse attention over ragged index sets: items ordered longest-first (lpt_order).  The
    // block path clears it for its own top-k sets (every count == k: nothing to balance).
    bool lpt = true;

    // Workspace slot of at least `bytes`; `s` (the calling op's stream) lets a growth during
    // stream capture fail loudly instead of allocating inside the capture.
    void* ws(int slot, size_t bytes, cudaStream_t s = nullptr);
    cublasHandle_t blas();
};

csd_status set_error(csd_status s, const char* fmt, ...);
csd_status cuda_status(cudaError_t e, const char* where);
csd_status check_flags(Ctx* ctx, cudaStream_t s);
csd_status gemm_bf16(Ctx* ctx, const void* a, const void* b, bool b_nk, void* c, bool c_f32,
                     int64_t m, int64_t n, int64_t k, float beta, cudaStream_t s);
csd_status gemm_bf16_chunks(Ctx* ctx, const void* cm, const void* w2, void* out, bool c_f32,
                            int64_t chunks, int64_t chunk, int64_t d, int64_t f, cudaStream_t s);
csd_status prod_dense_mlp(Ctx* c, const void* x, const void* w1, const float* b1, const void* w2,
                          const float* b2, int64_t batch, int64_t n, int64_t d, int64_t f,
                          int64_t chunk, float* out, void* act_cm, const void* x_mid, void* x_out,
                          cudaStream_t s);

}  // namespace csd
