// The production route behind the reference C++ API (include/csd/device.hpp) as a reference
// caller uses it: csd::dev:: ops and DeviceModel against the CHECK-mode csd:: functions
// (bit-exact with the reference), relative L2 <= 2e-2 (north_star's bf16 tolerance).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "csd/attention.hpp"
#include "csd/device.hpp"
#include "csd/mlp.hpp"
#include "csd/model.hpp"
#include "csd/rng.hpp"

static double rel(const csd::Tensor& a, const csd::Tensor& b, const csd::Tensor* base = nullptr) {
    double num = 0, den = 0;
    for (int64_t i = 0; i < a.numel(); ++i) {
        const double r = b[i] - (base ? (*base)[i] : 0.0);
        num += (a[i] - b[i]) * (a[i] - b[i]);
        den += r * r;
    }
    return std::sqrt(num / (den > 0 ? den : 1e-30));
}

// round to the nearest bf16 value (what the PROD path stores), ties to even
static void round_bf16(csd::Tensor& t) {
    for (int64_t i = 0; i < t.numel(); ++i) {
        uint32_t u;
        std::memcpy(&u, &t[i], 4);
        u += 0x7fffu + ((u >> 16) & 1u);
        u &= 0xffff0000u;
        std::memcpy(&t[i], &u, 4);
    }
}

static csd::Tensor randn(csd::GaussianRng& rng, std::vector<int64_t> shape, float s) {
    csd::Tensor t(std::move(shape));
    for (int64_t i = 0; i < t.numel(); ++i) t[i] = rng.next(0.0f, s);
    return t;
}

#define EXPECT(cond, ...)                          \
    do {                                           \
        if (!(cond)) {                             \
            std::printf("FAILED: " __VA_ARGS__);   \
            std::printf("\n");                     \
            return 1;                              \
        }                                          \
    } while (0)

int main() {
    csd::GaussianRng rng(7);
    // ---- attention ops, [B, H, N, E] = [1, 2, 512, 64], chunk 64
    const int64_t B = 1, H = 2, N = 512, E = 64, c = 64, k = 52;
    const auto q = randn(rng, {B, H, N, E}, 1.0f), kk = randn(rng, {B, H, N, E}, 1.0f),
               v = randn(rng, {B, H, N, E}, 1.0f), base = randn(rng, {B, H, N, E}, 1.0f);
    const double e_dense = rel(csd::dev::dense_attention(q, kk, v), csd::dense_attention(q, kk, v));
    EXPECT(e_dense < 2e-2, "dense_attention rel %.3g", e_dense);
    const auto cs_ref = csd::column_sum_attention(q, kk, v, nullptr, c);
    const auto cs = csd::dev::column_sum_attention(q, kk, v, nullptr, c);
    EXPECT(rel(cs.output, cs_ref.output) < 2e-2, "column_sum_attention output");
    EXPECT(rel(cs.column_sums, cs_ref.column_sums) < 2e-2, "column sums %.3g",
           rel(cs.column_sums, cs_ref.column_sums));
    const auto idx = csd::select_top_k(cs_ref.column_sums, k, c);
    const double e_sp = rel(csd::dev::sparse_delta_attention(q, kk, v, idx, base, 1.0f),
                            csd::sparse_delta_attention(q, kk, v, idx, base, 1.0f), &base);
    EXPECT(e_sp < 2e-2, "sparse_delta_attention rel %.3g", e_sp);
    bool threw = false;
    try {  // the reference's error types: an index set of the wrong shape
        csd::dev::sparse_delta_attention(q, kk, v, csd::SparseIndexSet::empty(1, 3, N / c, c, k, N), base, 1.0f);
    } catch (const csd::ShapeError&) {
        threw = true;
    }
    EXPECT(threw, "ShapeError expected");

    // ---- MLP ops, D 256, F 1024, chunk 64
    const int64_t D = 256, F = 1024;
    csd::MlpWeights w;
    w.w1 = randn(rng, {F, D}, 1.0f / 16);
    w.b1 = randn(rng, {F}, 0.1f);
    w.w2 = randn(rng, {F, D}, 0.5f / 16);
    w.b2 = randn(rng, {D}, 0.1f);
    const auto x = randn(rng, {1, N, D}, 1.0f);
    const auto dm = csd::dev::dense_mlp(x, w, c);
    const auto dm_ref = csd::dense_mlp(x, w);
    EXPECT(rel(dm.output, dm_ref.output) < 2e-2, "dense_mlp output %.3g", rel(dm.output, dm_ref.output));
    EXPECT(rel(dm.act, dm_ref.act) < 2e-2, "dense_mlp act");
    const auto tm = csd::dev::mlp_tile_means(x, w.w1, c);
    EXPECT(rel(tm, csd::mlp_tile_means(x, w.w1, c)) < 1e-2, "mlp_tile_means");

    // ---- DeviceModel vs model_forward_step (CHECK), 2 layers, D S S D S, outputs fed back
    csd::ModelConfig cfg;
    cfg.grid_t = 1;
    cfg.grid_h = 32;
    cfg.grid_w = 32;
    cfg.voxel_t = 1;
    cfg.voxel_h = 8;
    cfg.voxel_w = 8;
    cfg.chunk = 64;
    cfg.model_dim = 256;
    cfg.heads = 4;
    cfg.head_dim = 64;
    cfg.mlp_hidden = 1024;
    cfg.layers = 2;
    auto model = csd::build_toy_model(cfg);
    // both paths see the same bf16-representable weights and inputs (the PROD storage),
    // so the comparison measures the arithmetic, as the north_star tolerance means it
    for (auto& lw : model.layers)
        for (csd::Tensor* t : {&lw.wq, &lw.wk, &lw.wv, &lw.wo, &lw.mlp.w1, &lw.mlp.w2}) round_bf16(*t);
    const csd::SparsityConfig sp{102, 307};
    auto state = csd::make_state(model);
    csd::dev::DeviceModel dmod(model, sp);
    csd::Tensor xs = randn(rng, {1, cfg.seq_len(), cfg.model_dim}, 1.0f);
    const bool sched[] = {true, false, false, true, false};
    for (int t = 0; t < 5; ++t) {
        round_bf16(xs);
        const auto yr = csd::model_forward_step(model, state, xs, sched[t], sp);
        const auto yd = dmod.forward_step(xs, sched[t]);
        const double e = rel(yd, yr, &xs);
        std::printf("step %d (%s): rel L2 over the block branch %.3g\n", t, sched[t] ? "dense" : "sparse", e);
        EXPECT(e < 2e-2, "DeviceModel step %d rel %.3g", t, e);
        // the reference harness's latent update x <- x + y / T (harness.cpp:200, T = 50) on
        // the CHECK trajectory drives both paths
        for (int64_t i = 0; i < xs.numel(); ++i) xs[i] += yr[i] * (1.0f / 50.0f);
    }
    threw = false;
    try {
        dmod.reset();
        dmod.forward_step(xs, false);  // sparse step on a fresh state -> StateError
    } catch (const csd::StateError&) {
        threw = true;
    }
    EXPECT(threw, "StateError expected after reset");
    std::printf("device api tests passed\n");
    return 0;
}
