// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library, compiled from
// /root/reference/proj/src/*.cpp by oracle/Makefile with -Dcsd=csd_ref (the
// macro renames the namespace so the reference can sit beside our own csd::
// host mirror in one process).  Output: oracle/_ref/libcsd_ref.so.
//
// Used to (1) generate the golden fixtures under tests/golden/ (gen_golden.py),
// (2) cross-check the plain-C oracle in tests/test_oracle.py, and (3) time the
// reference CPU path in bench.py --impl reference.  Every entry point copies
// raw row-major buffers into csd_ref::Tensor, calls the reference function
// named in its comment, and copies the result out.  Exceptions are mapped to
// the same negative codes as oracle/csd_oracle.h.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <unistd.h>
#include <vector>

#include "csd/attention.hpp"
#include "csd/error.hpp"
#include "csd/harness.hpp"
#include "csd/mlp.hpp"
#include "csd/schedule.hpp"
#include "csd/tensor_io.hpp"
#include "csd/model.hpp"
#include "csd/rng.hpp"
#include "csd/sparse_index.hpp"
#include "csd/tensor.hpp"
#include "csd/voxel.hpp"

using namespace csd_ref;

namespace {

Tensor make(const float* p, std::vector<int64_t> shape) {
    int64_t n = 1;
    for (auto d : shape) n *= d;
    return Tensor(std::move(shape), std::vector<float>(p, p + n));
}

void put(const Tensor& t, float* out) {
    std::memcpy(out, t.data(), sizeof(float) * static_cast<size_t>(t.numel()));
}

SparseIndexSet make_set(const int32_t* idx, const int32_t* counts, int64_t batch, int64_t heads,
                        int64_t chunks, int64_t chunk, int64_t k_max, int64_t domain) {
    SparseIndexSet s = SparseIndexSet::empty(batch, heads, chunks, chunk, k_max, domain);
    std::memcpy(s.indices.data(), idx, sizeof(int32_t) * s.indices.size());
    std::memcpy(s.counts.data(), counts, sizeof(int32_t) * s.counts.size());
    return s;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError&) {
        return -1;
    } catch (const IndexError&) {
        return -2;
    } catch (const NumericError&) {
        return -3;
    } catch (const StateError&) {
        return -4;
    } catch (const ValueError&) {
        return -5;
    } catch (const ConfigError&) {
        return -6;
    } catch (const std::exception&) {
        return -100;
    }
}

}  // namespace

extern "C" {

// rng.hpp:12-44 via tests/test_util.hpp:50-55 (random_tensor).
void ref_gaussian(uint64_t seed, int64_t n, float stddev, float* out) {
    GaussianRng rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng.next(0.0f, stddev);
}

// voxel.cpp:18-42
int ref_voxel_permutation(int64_t t, int64_t h, int64_t w, int64_t vt, int64_t vh, int64_t vw,
                          int64_t* perm) {
    return guard([&] {
        auto p = voxel_permutation(VoxelLayout{t, h, w, vt, vh, vw});
        std::memcpy(perm, p.data(), sizeof(int64_t) * p.size());
    });
}

// voxel.cpp:44-73
int ref_voxel_order(const float* x, int64_t b, int64_t t, int64_t h, int64_t w, int64_t d,
                    int64_t vt, int64_t vh, int64_t vw, float* out) {
    return guard([&] {
        auto r = voxel_order(make(x, {b, t, h, w, d}), VoxelLayout{t, h, w, vt, vh, vw});
        put(r.reordered, out);
    });
}

// voxel.cpp:75-102
int ref_reverse_voxel_order(const float* x, int64_t b, int64_t t, int64_t h, int64_t w, int64_t d,
                            int64_t vt, int64_t vh, int64_t vw, float* out) {
    return guard([&] {
        put(reverse_voxel_order(make(x, {b, t * h * w, d}), VoxelLayout{t, h, w, vt, vh, vw}), out);
    });
}

// sparse_index.cpp:64-96 (scores viewed as [1, 1, rows, m])
int ref_select_top_k(const float* scores, int64_t rows, int64_t m, int64_t k, int32_t* idx) {
    return guard([&] {
        auto s = select_top_k(make(scores, {1, 1, rows, m}), k, 1);
        std::memcpy(idx, s.indices.data(), sizeof(int32_t) * s.indices.size());
    });
}

// attention.cpp:59-74
int ref_dense_attention(const float* q, const float* k, const float* v, int64_t b, int64_t h,
                        int64_t n, int64_t e, float* out) {
    return guard([&] {
        put(dense_attention(make(q, {b, h, n, e}), make(k, {b, h, n, e}), make(v, {b, h, n, e})),
            out);
    });
}

// attention.cpp:76-145
int ref_column_sum_attention(const float* q, const float* k, const float* v, const float* prev_m,
                             const float* prev_l, int64_t b, int64_t h, int64_t n, int64_t e,
                             int64_t chunk, float* out, float* row_max, float* exp_sum,
                             float* colsum) {
    return guard([&] {
        SoftmaxStats prev;
        const SoftmaxStats* pp = nullptr;
        if (prev_m != nullptr) {
            prev.row_max = make(prev_m, {b, h, n});
            prev.exp_sum = make(prev_l, {b, h, n});
            pp = &prev;
        }
        auto r = column_sum_attention(make(q, {b, h, n, e}), make(k, {b, h, n, e}),
                                      make(v, {b, h, n, e}), pp, chunk);
        put(r.output, out);
        put(r.stats.row_max, row_max);
        put(r.stats.exp_sum, exp_sum);
        put(r.column_sums, colsum);
    });
}

// attention.cpp:147-194
int ref_sparse_delta_attention(const float* q, const float* k, const float* v, const int32_t* idx,
                               const int32_t* counts, int64_t k_max, int64_t chunk,
                               const float* base, float scale, int64_t b, int64_t h, int64_t n,
                               int64_t e, float* out) {
    return guard([&] {
        auto set = make_set(idx, counts, b, h, n / chunk, chunk, k_max, n);
        put(sparse_delta_attention(make(q, {b, h, n, e}), make(k, {b, h, n, e}),
                                   make(v, {b, h, n, e}), set, make(base, {b, h, n, e}), scale),
            out);
    });
}

static MlpWeights make_w(const float* w1, const float* b1, const float* w2, const float* b2,
                         int64_t d, int64_t f) {
    MlpWeights w;
    w.w1 = make(w1, {f, d});
    w.b1 = make(b1, {f});
    w.w2 = make(w2, {f, d});
    w.b2 = make(b2, {d});
    return w;
}

// mlp.cpp:49-81
int ref_dense_mlp(const float* x, const float* w1, const float* b1, const float* w2,
                  const float* b2, int64_t b, int64_t n, int64_t d, int64_t f, float* out,
                  float* pre, float* act) {
    return guard([&] {
        auto r = dense_mlp(make(x, {b, n, d}), make_w(w1, b1, w2, b2, d, f));
        put(r.output, out);
        if (pre) put(r.preact, pre);
        if (act) put(r.act, act);
    });
}

// mlp.cpp:83-96
int ref_mlp_tile_means(const float* x, const float* w1, int64_t b, int64_t n, int64_t d, int64_t f,
                       int64_t chunk, float* out) {
    return guard([&] { put(mlp_tile_means(make(x, {b, n, d}), make(w1, {f, d}), chunk), out); });
}

// mlp.cpp:98-118
int ref_mlp_change_indices(const float* x, const float* w1, const float* tile_means, int64_t b,
                           int64_t n, int64_t d, int64_t f, int64_t k, int64_t chunk,
                           int32_t* idx) {
    return guard([&] {
        auto s = mlp_change_indices(make(x, {b, n, d}), make(w1, {f, d}),
                                    make(tile_means, {b, n / chunk, f}), k, chunk);
        std::memcpy(idx, s.indices.data(), sizeof(int32_t) * s.indices.size());
    });
}

// mlp.cpp:120-182 (cache arrays updated in place, like MlpCache)
int ref_sparse_delta_mlp(const float* x, const float* w1, const float* b1, const float* w2,
                         const float* b2, const int32_t* idx, const int32_t* counts,
                         int64_t k_max, int64_t chunk, int64_t b, int64_t n, int64_t d, int64_t f,
                         float* act_cache, float* out_cache) {
    return guard([&] {
        MlpCache cache;
        cache.activations = make(act_cache, {b, n, f});
        cache.outputs = make(out_cache, {b, n, d});
        cache.initialized = true;
        auto set = make_set(idx, counts, b, 1, n / chunk, chunk, k_max, f);
        sparse_delta_mlp(make(x, {b, n, d}), make_w(w1, b1, w2, b2, d, f), set, cache);
        put(cache.activations, act_cache);
        put(cache.outputs, out_cache);
    });
}

// ---------------------------------------------------------------------------
// Block level (model.cpp:79-99, :167-216): a toy model held behind an opaque
// handle so golden block trajectories and the CPU baseline can be produced.
struct RefModel {
    ToyModel model;
    ModelState state;
};

void* ref_model_create(int64_t batch, int64_t gt, int64_t gh, int64_t gw, int64_t d, int64_t e,
                       int64_t heads, int64_t f, int64_t layers, int64_t vt, int64_t vh,
                       int64_t vw, int64_t chunk, uint64_t seed) {
    try {
        ModelConfig cfg;
        cfg.batch = batch; cfg.grid_t = gt; cfg.grid_h = gh; cfg.grid_w = gw;
        cfg.model_dim = d; cfg.head_dim = e; cfg.heads = heads; cfg.mlp_hidden = f;
        cfg.layers = layers; cfg.voxel_t = vt; cfg.voxel_h = vh; cfg.voxel_w = vw;
        cfg.chunk = chunk; cfg.seed = seed;
        auto* m = new RefModel;
        m->model = build_toy_model(cfg);
        m->state = make_state(m->model);
        return m;
    } catch (...) {
        return nullptr;
    }
}

void ref_model_destroy(void* h) { delete static_cast<RefModel*>(h); }

// Weights of layer l in reference layout: which = 0..7 -> wq wk wv wo w1 b1 w2 b2.
int ref_model_weight(void* h, int64_t layer, int which, float* out) {
    auto* m = static_cast<RefModel*>(h);
    const auto& lw = m->model.layers.at(static_cast<size_t>(layer));
    const Tensor* t[] = {&lw.wq, &lw.wk, &lw.wv, &lw.wo, &lw.mlp.w1, &lw.mlp.b1, &lw.mlp.w2,
                         &lw.mlp.b2};
    put(*t[which], out);
    return 0;
}

// model.cpp:178-216
int ref_model_step(void* h, const float* x, int dense, int64_t attn_k, int64_t mlp_k,
                   float* out) {
    auto* m = static_cast<RefModel*>(h);
    return guard([&] {
        const auto& c = m->model.cfg;
        SparsityConfig sp;
        sp.attn_k = attn_k;
        sp.mlp_k = mlp_k;
        put(model_forward_step(m->model, m->state, make(x, {c.batch, c.seq_len(), c.model_dim}),
                               dense != 0, sp),
            out);
    });
}

// model.cpp:178-216 with a static attention pattern (model.hpp:97-99, attention.hpp:50-52):
// idx [B, H, C, k_max] / counts [B, H, C] replace the top-k on dense steps, verbatim.
int ref_model_step_static(void* h, const float* x, int dense, int64_t attn_k, int64_t mlp_k,
                          const int32_t* idx, const int32_t* counts, int64_t k_max, float* out) {
    auto* m = static_cast<RefModel*>(h);
    return guard([&] {
        const auto& c = m->model.cfg;
        SparsityConfig sp;
        sp.attn_k = attn_k;
        sp.mlp_k = mlp_k;
        const int64_t chunks = c.seq_len() / c.chunk;
        const SparseIndexSet st =
            make_set(idx, counts, c.batch, c.heads, chunks, c.chunk, k_max, c.seq_len());
        put(model_forward_step(m->model, m->state, make(x, {c.batch, c.seq_len(), c.model_dim}),
                               dense != 0, sp, nullptr, &st),
            out);
    });
}

// model.cpp:167-176
int ref_model_dense(void* h, const float* x, float* out) {
    auto* m = static_cast<RefModel*>(h);
    return guard([&] {
        const auto& c = m->model.cfg;
        put(model_forward_dense(m->model, make(x, {c.batch, c.seq_len(), c.model_dim})), out);
    });
}

// Per-layer cache views after a step (reference layouts), for parity tests.
// which: 0 attn residual [B,H,N,E], 1 row_max [B,H,N], 2 exp_sum, 3 mlp act [B,N,F],
// 4 mlp out [B,N,D], 5 mlp tile means [B,C,F].
int ref_model_cache(void* h, int64_t layer, int which, float* out) {
    auto* m = static_cast<RefModel*>(h);
    const auto& ls = m->state.layers.at(static_cast<size_t>(layer));
    const Tensor* t[] = {&ls.attn.residual_output, &ls.attn.stats.row_max, &ls.attn.stats.exp_sum,
                         &ls.mlp.activations, &ls.mlp.outputs, &ls.mlp.tile_means};
    put(*t[which], out);
    return 0;
}

// Index sets after a step: attention [B,H,C,k] (k_max from cache) or MLP [B,1,C,k].
int ref_model_indices(void* h, int64_t layer, int mlp, int32_t* idx, int32_t* counts) {
    auto* m = static_cast<RefModel*>(h);
    const auto& ls = m->state.layers.at(static_cast<size_t>(layer));
    const SparseIndexSet& s = mlp ? ls.mlp.indices : ls.attn.indices;
    std::memcpy(idx, s.indices.data(), sizeof(int32_t) * s.indices.size());
    std::memcpy(counts, s.counts.data(), sizeof(int32_t) * s.counts.size());
    return static_cast<int>(s.k_max);
}


// schedule.cpp:44-87 -> modes[total_steps] (0 dense, 1 sparse, 2 skipped)
int ref_resolve_schedule(int64_t total_steps, int64_t dense_interval, int step_cache,
                         int64_t window, int64_t stride, int32_t* modes) {
    return guard([&] {
        const StepSchedule s = resolve_schedule(total_steps, dense_interval, step_cache != 0,
                                                window, stride);
        for (int64_t i = 0; i < total_steps; ++i)
            modes[i] = static_cast<int32_t>(s.modes[static_cast<size_t>(i)]);
    });
}

// harness.cpp:123-224 (run_generation, RunMode::SparseDelta): the seeded toy model and
// latent of `cfg`, the resolved schedule, x += (1/T) * model output per step (skipped steps
// reuse the last output), latent R^2 vs the dense trajectory per step.  Outputs: modes,
// per-step latent R^2 (NaN when undefined), end-to-end R^2, and the decoded final latent
// [B, T, H, W, D] (read back from the reference's own CSDT dump, tensor_io.cpp).
// cfg = {batch, grid_t, grid_h, grid_w, dim, head_dim, heads, hidden, layers, voxel_t,
//        voxel_h, voxel_w, chunk, seed}; sch = {total_steps, dense_interval, step_cache,
//        window, stride, attn_k, mlp_k}
int ref_run_generation(const int64_t* cfg, const int64_t* sch, int32_t* modes, double* latent_r2,
                       double* e2e_r2, float* final_latent) {
    return guard([&] {
        RunRequest req;
        ModelConfig& m = req.model;
        m.batch = cfg[0]; m.grid_t = cfg[1]; m.grid_h = cfg[2]; m.grid_w = cfg[3];
        m.model_dim = cfg[4]; m.head_dim = cfg[5]; m.heads = cfg[6]; m.mlp_hidden = cfg[7];
        m.layers = cfg[8]; m.voxel_t = cfg[9]; m.voxel_h = cfg[10]; m.voxel_w = cfg[11];
        m.chunk = cfg[12]; m.seed = static_cast<uint64_t>(cfg[13]);
        req.schedule.total_steps = sch[0];
        req.schedule.dense_interval = sch[1];
        req.schedule.step_cache = sch[2] != 0;
        req.schedule.window = sch[3];
        req.schedule.stride = sch[4];
        req.sparsity.attn_k = sch[5];
        req.sparsity.mlp_k = sch[6];
        req.mode = RunMode::SparseDelta;
        char path[] = "/tmp/csd_ref_latent_XXXXXX";
        const int fd = mkstemp(path);
        if (fd >= 0) close(fd);
        req.save_latent_path = path;
        const RunReport rep = run_generation(req);
        for (size_t i = 0; i < rep.steps.size(); ++i) {
            modes[i] = static_cast<int32_t>(rep.steps[i].mode);
            latent_r2[i] = rep.steps[i].latent_r2.value_or(std::nan(""));
        }
        *e2e_r2 = rep.end_to_end_r2.value_or(std::nan(""));
        put(load_tensor(std::string(path)), final_latent);
        std::remove(path);
    });
}

}  // extern "C"
