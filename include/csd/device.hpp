// device.hpp — the PRODUCTION route behind the reference's C++ API.
//
// The csd:: functions of attention.hpp / mlp.hpp / model.hpp (libcsd_host.so) run in CHECK
// mode: fp32 CUDA-core kernels, bit-exact with the reference.  csd::dev:: offers the same
// operations in PROD mode -- bf16 storage, fp32 accumulation, the tcgen05 kernels -- with the
// reference's argument meaning, validation and exception types, and results within the
// north_star tolerance (relative L2 <= 2e-2) instead of bit-exact:
//
//   * the stateless attention / MLP ops (attention.hpp:27-52, mlp.hpp:33-65) on host
//     tensors: inputs are rounded to bf16 on the device, outputs come back as fp32;
//   * DeviceModel: model_forward_step (model.cpp:178-216) with every layer's weights and
//     caches resident on the B200 between steps (csd_block_* per layer) -- the path a
//     reference caller uses for speed, with a device-pointer entry for callers that keep
//     their latent on the GPU.
#pragma once

#include <cstdint>
#include <vector>

#include "csd/attention.hpp"
#include "csd/mlp.hpp"
#include "csd/model.hpp"

namespace csd {
namespace dev {

// attention.cpp:59-74 / :76-145 / :147-194 on the tcgen05 kernels ([B, H, N, E] tensors)
Tensor dense_attention(const Tensor& q, const Tensor& k, const Tensor& v);
ColumnSumAttentionResult column_sum_attention(const Tensor& q, const Tensor& k, const Tensor& v,
                                              const SoftmaxStats* prev_stats, int64_t chunk);
Tensor sparse_delta_attention(const Tensor& q, const Tensor& k, const Tensor& v,
                              const SparseIndexSet& indices, const Tensor& base, float scale);

// mlp.cpp:49-81 / :83-96 / :98-118 (output and the activations in the reference layout;
// preact is not materialised by the fused GEMM and comes back empty)
MlpDenseResult dense_mlp(const Tensor& x, const MlpWeights& w, int64_t chunk);
Tensor mlp_tile_means(const Tensor& x, const Tensor& w1, int64_t chunk);
SparseIndexSet mlp_change_indices(const Tensor& x, const Tensor& w1, const Tensor& tile_means,
                                  int64_t k, int64_t chunk);

// model_forward_step for a whole ToyModel on the device (one csd_block per layer).
class DeviceModel {
public:
    DeviceModel(const ToyModel& model, const SparsityConfig& sparsity);
    ~DeviceModel();
    DeviceModel(const DeviceModel&) = delete;
    DeviceModel& operator=(const DeviceModel&) = delete;

    // x, result: host fp32 [B, N, D] (the reference's signature, minus the probe)
    Tensor forward_step(const Tensor& x, bool dense_step, const SparseIndexSet* static_attn = nullptr);
    // x_bf16 / y_bf16: device bf16 [B, N, D]; stream: a cudaStream_t (nullptr = default)
    void forward_step_device(const void* x_bf16, void* y_bf16, bool dense_step, void* stream);
    void reset();  // make_state: every cache empty, the next step must be dense
    int64_t layers() const { return static_cast<int64_t>(blocks_.size()); }

private:
    ModelConfig cfg_;
    SparsityConfig sparsity_;
    std::vector<void*> blocks_;  // csd_block*
    void* buf_[2] = {nullptr, nullptr};  // layer ping-pong activations (bf16)
    void* io_ = nullptr;                 // fp32 staging for host tensors
};

}  // namespace dev
}  // namespace csd
