// Drives the block-stack API (include/csd/model.hpp, libcsd_host.so) the way a reference
// caller would (harness.cpp:186-212): build_toy_model -> make_state -> model_forward_step
// over a dense/sparse schedule, plus model_forward_dense.  Writes the outputs as raw fp32 to
// argv[1] for tests/test_model_mirror.py to compare with the reference library.
#include <cstdio>
#include <vector>

#include "csd/model.hpp"
#include "csd/rng.hpp"

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    csd::ModelConfig cfg;  // reference defaults: 2 layers, grid 2x8x8, D 64, 4x16, F 128, c 4
    const auto model = csd::build_toy_model(cfg);
    auto state = csd::make_state(model);
    csd::GaussianRng rng(cfg.seed + 1);
    csd::Tensor x({cfg.batch, cfg.seq_len(), cfg.model_dim});
    for (int64_t i = 0; i < x.numel(); ++i) x[i] = rng.next(0.0f, 1.0f);
    const csd::SparsityConfig sp{8, 32};
    std::FILE* f = std::fopen(argv[1], "wb");
    const bool sched[] = {true, false, false, true, false};
    csd::Tensor cur = x;
    for (bool dense : sched) {
        cur = csd::model_forward_step(model, state, cur, dense, sp);
        std::fwrite(cur.data(), sizeof(float), cur.numel(), f);
    }
    const csd::Tensor d = csd::model_forward_dense(model, x);
    std::fwrite(d.data(), sizeof(float), d.numel(), f);
    std::fclose(f);
    try {  // sparse before dense on a fresh state -> StateError (model.cpp via attention.cpp:199)
        auto fresh = csd::make_state(model);
        csd::model_forward_step(model, fresh, x, false, sp);
        return 3;
    } catch (const csd::StateError&) {
    }
    return 0;
}
