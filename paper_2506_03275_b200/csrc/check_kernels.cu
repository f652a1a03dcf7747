// check_kernels.cu — CSD_MODE_CHECK kernels: fp32, bit-exact reproduction of
// the reference arithmetic (compiled with -fmad=false; every float op is an
// explicit round-to-nearest intrinsic in the reference's order).
//
// The core is one tiled "sequential-k" GEMM: each thread owns one output and
// accumulates k in increasing order exactly like tensor.cpp:83-96
// (acc = 0; acc += a*b), so shared-memory tiling changes nothing but speed.
// Gathers (K_S, V_S, W1[S], W2[S]) are folded into the B-operand load.
#include <cuda_runtime.h>

#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace csd {
namespace dev {

constexpr int TS = 16;  // output tile edge and k-tile depth

// Batched problem descriptor.  Batch z covers `rows` rows of A starting at
// a_off(z); its B operand rows are gathered through idx (or identity).
struct ExactGemm {
    // A: element (m, k) = a[a_base + m*lda + k]
    const float* a;
    int64_t lda;
    // B: trans -> element (k, n) = b[b_base + row(n)*ldb + k]   (x @ W^T)
    //    !trans -> element (k, n) = b[b_base + row(k)*ldb + n]  (P @ V)
    const float* b;
    int64_t ldb;
    bool trans_b;
    // C: element (m, n) = c[c_base + m*ldc + n]
    float* c;
    int64_t ldc;
    int64_t M, N, K;  // maxima; per-batch counts may shrink N (trans) or K (!trans)
    const int32_t* idx;     // gather list per batch (nullable = identity)
    const int32_t* counts;  // per-batch active length (nullable = full)
    int64_t idx_stride;     // k_max
    // Batch z -> base offsets: off = (z / inner) * outer_stride + (z % inner) * inner_stride
    int64_t inner;
    int64_t a_os, a_is, b_os, b_is, c_os, c_is;
    // epilogue
    int epi;         // 0 store, 1 scale, 2 bias(+n)->store, 3 bias+gelu, 4 c += acc, 5 c = base + s*acc
    float scale;
    const float* bias;  // epi 2/3: bias[row_of(n)]  epi 5: base with same addressing as c
    int64_t base_off_extra;
};

__device__ __forceinline__ int64_t boff(int64_t z, int64_t inner, int64_t os, int64_t is) {
    return (z / inner) * os + (z % inner) * is;
}

__global__ void k_exact_gemm(ExactGemm p) {
    __shared__ float As[TS][TS + 1];
    __shared__ float Bs[TS][TS + 1];
    const int64_t z = blockIdx.z;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t m = (int64_t)blockIdx.y * TS + ty;
    const int64_t n = (int64_t)blockIdx.x * TS + tx;
    const int64_t cnt = p.counts ? p.counts[z] : (p.trans_b ? p.N : p.K);
    const int64_t Nz = p.trans_b ? cnt : p.N;
    const int64_t Kz = p.trans_b ? p.K : cnt;
    if (cnt == 0) return;
    if ((int64_t)blockIdx.x * TS >= Nz || (int64_t)blockIdx.y * TS >= p.M) return;
    const float* a = p.a + boff(z, p.inner, p.a_os, p.a_is);
    const float* b = p.b + boff(z, p.inner, p.b_os, p.b_is);
    const int32_t* idx = p.idx ? p.idx + z * p.idx_stride : nullptr;
    float acc = 0.0f;
    for (int64_t k0 = 0; k0 < Kz; k0 += TS) {
        // A tile: rows m0..m0+15, k0..k0+15
        {
            const int64_t am = (int64_t)blockIdx.y * TS + ty, ak = k0 + tx;
            As[ty][tx] = (am < p.M && ak < Kz) ? a[am * p.lda + ak] : 0.0f;
        }
        // B tile as Bs[k][n]
        if (p.trans_b) {
            const int64_t bn = (int64_t)blockIdx.x * TS + ty, bk = k0 + tx;
            float v = 0.0f;
            if (bn < Nz && bk < Kz) {
                const int64_t row = idx ? idx[bn] : bn;
                v = b[row * p.ldb + bk];
            }
            Bs[tx][ty] = v;
        } else {
            const int64_t bk = k0 + ty, bn = (int64_t)blockIdx.x * TS + tx;
            float v = 0.0f;
            if (bn < Nz && bk < Kz) {
                const int64_t row = idx ? idx[bk] : bk;
                v = b[row * p.ldb + bn];
            }
            Bs[ty][tx] = v;
        }
        __syncthreads();
        const int64_t kend = (Kz - k0) < TS ? (Kz - k0) : TS;
        for (int kk = 0; kk < kend; ++kk) acc = __fadd_rn(acc, __fmul_rn(As[ty][kk], Bs[kk][tx]));
        __syncthreads();
    }
    if (m >= p.M || n >= Nz) return;
    float* c = p.c + boff(z, p.inner, p.c_os, p.c_is) + m * p.ldc + n;
    switch (p.epi) {
        case 0: *c = acc; break;
        case 1: *c = __fmul_rn(acc, p.scale); break;
        case 2: {
            const int64_t row = idx ? idx[n] : n;
            *c = __fadd_rn(acc, p.bias[row]);
        } break;
        case 3: {
            const int64_t row = idx ? idx[n] : n;
            *c = exact_gelu(__fadd_rn(acc, p.bias[row]));
        } break;
        case 4: *c = __fadd_rn(*c, acc); break;
        case 5: {
            const float* base = p.bias + boff(z, p.inner, p.c_os, p.c_is) + m * p.ldc + n;
            *c = __fadd_rn(*base, __fmul_rn(p.scale, acc));
        } break;
    }
}

static cudaError_t launch_exact(const ExactGemm& p, int64_t batches, cudaStream_t s) {
    const int64_t nt = p.trans_b ? p.N : p.N;
    dim3 grid((unsigned)((nt + TS - 1) / TS), (unsigned)((p.M + TS - 1) / TS), (unsigned)batches);
    k_exact_gemm<<<grid, dim3(TS, TS), 0, s>>>(p);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Row softmax over the first cnt entries of each row (tensor.cpp:100-139):
// m = row max (std::max order), l = sequential sum of expf(x - m), probs /= l.
// rows are grouped: row r belongs to batch r / rows_per_batch.
__global__ void k_softmax_rows(float* buf, int64_t rows, int64_t rows_per_batch, int64_t stride,
                               const int32_t* counts, int64_t full, float* row_max,
                               float* exp_sum, uint32_t* flags) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int64_t cnt = counts ? counts[r / rows_per_batch] : full;
    if (cnt == 0) return;
    float* row = buf + r * stride;
    float m = row[0];
    for (int64_t j = 0; j < cnt; ++j) {
        const float x = row[j];
        if (!isfinite(x)) raise_flag(flags, kFlagNonFinite);
        m = (m < x) ? x : m;
    }
    float l = 0.0f;
    for (int64_t j = 0; j < cnt; ++j) {
        const float e = exact_expf(__fsub_rn(row[j], m));
        row[j] = e;
        l = __fadd_rn(l, e);
    }
    for (int64_t j = 0; j < cnt; ++j) row[j] = __fdiv_rn(row[j], l);
    if (row_max) row_max[r] = m;
    if (exp_sum) exp_sum[r] = l;
}

// Column sums with (possibly stale) stats (attention.cpp:128-138):
// cs[bh, c, j] = sum_{i in chunk c} expf(L[i, j] - m[i]) / l[i], i ascending.
__global__ void k_colsum_exact(const float* logits, const float* m, const float* l, int64_t n,
                               int64_t chunk, int64_t bh_count, float* out) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t c = blockIdx.y;
    const int64_t bh = blockIdx.z;
    if (j >= n || bh >= bh_count) return;
    const float* L = logits + bh * n * n;
    const float* mm = m + bh * n;
    const float* ll = l + bh * n;
    float w = 0.0f;
    for (int64_t i = c * chunk; i < (c + 1) * chunk; ++i)
        w = __fadd_rn(w, __fdiv_rn(exact_expf(__fsub_rn(L[i * n + j], mm[i])), ll[i]));
    out[(bh * (n / chunk) + c) * n + j] = w;
}

// chunk_reduce Mean (tensor.cpp:208-221): w = 0; w += row (rows in order); w *= 1/c.
__global__ void k_chunk_mean_exact(const float* x, int64_t batch, int64_t n, int64_t d,
                                   int64_t chunk, float* out) {
    const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t bc = blockIdx.y;  // b * C + c
    const int64_t nc = n / chunk;
    if (col >= d || bc >= batch * nc) return;
    const int64_t b = bc / nc, c = bc % nc;
    const float inv = __fdiv_rn(1.0f, (float)chunk);
    float w = 0.0f;
    for (int64_t r = c * chunk; r < (c + 1) * chunk; ++r) w = __fadd_rn(w, x[(b * n + r) * d + col]);
    out[bc * d + col] = __fmul_rn(w, inv);
}

__global__ void k_absdiff(const float* a, const float* b, int64_t n, float* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = fabsf(__fsub_rn(a[i], b[i]));
}

__global__ void k_add_exact(const float* a, const float* b, int64_t n, float* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = __fadd_rn(a[i], b[i]);
}

// Sparse MLP activation refresh (mlp.cpp:153-171): for selected neuron j of
// chunk z: fresh = gelu(pre + b1) [pre from the exact GEMM, bias added by it],
// delta = fresh - A[row, f]; A[row, f] = fresh.  pre/delta share a buffer.
__global__ void k_mlp_refresh_exact(float* pre_delta, const int32_t* idx, const int32_t* counts,
                                    int64_t k_max, int64_t chunk, int64_t n, int64_t f,
                                    int64_t chunks_total, float* act_ref) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t rz = blockIdx.y;  // row within all chunks: z * chunk + r
    const int64_t z = rz / chunk, r = rz % chunk;
    if (z >= chunks_total) return;
    const int64_t cnt = counts[z];
    if (j >= cnt) return;
    const int64_t neuron = idx[z * k_max + j];
    float* pd = pre_delta + rz * k_max + j;
    const float fresh = *pd;  // already gelu'd by the GEMM epilogue
    // row in [B,N,F]: z = b*C + c -> token b*n + c*chunk + r
    const int64_t nc = n / chunk;
    const int64_t tok = (z / nc) * n + (z % nc) * chunk + r;
    float* cached = act_ref + tok * f + neuron;
    *pd = __fsub_rn(fresh, *cached);
    *cached = fresh;
}

// ---------------------------------------------------------------------------
// Host launchers.
static inline int64_t row_off(int layout, int64_t b, int64_t h, int64_t heads, int64_t n,
                              int64_t e) {
    // offset of token 0 of (b, h) and the row stride
    return layout == CSD_LAYOUT_BHNE ? ((b * heads + h) * n) * e : (b * n * heads + h) * e;
}

cudaError_t check_attention_logits(const float* q, const float* k, int layout, int64_t batch,
                                   int64_t heads, int64_t n, int64_t e, int64_t chunk,
                                   const int32_t* idx, const int32_t* counts, int64_t k_max,
                                   float* logits, cudaStream_t s) {
    // One batch per (b, h, chunk) when gathering; per (b, h) with identity.
    const int64_t rs = layout == CSD_LAYOUT_BHNE ? e : heads * e;  // token stride
    ExactGemm p{};
    p.trans_b = true;
    p.epi = 1;
    p.scale = 1.0f / std::sqrt((float)e);  // attention.cpp:40 (host IEEE sqrt + div)
    if (idx) {
        const int64_t nc = n / chunk;
        p.M = chunk; p.N = k_max; p.K = e;
        p.idx = idx; p.counts = counts; p.idx_stride = k_max;
        p.inner = nc;
        // batch z = bh * nc + c; A rows = tokens c*chunk.., B = k of (b,h)
        p.a = q; p.lda = rs; p.b = k; p.ldb = rs; p.c = logits; p.ldc = k_max;
        // offsets depend on (b, h) = z / nc: layout-specific linear in bh only if BHNE.
        // Use per-(b,h) launches for BNHE to keep the descriptor affine.
        if (layout == CSD_LAYOUT_BHNE) {
            p.a_os = n * e; p.a_is = chunk * e;
            p.b_os = n * e; p.b_is = 0;
            p.c_os = n * k_max; p.c_is = chunk * k_max;
            return launch_exact(p, batch * heads * nc, s);
        }
        for (int64_t b = 0; b < batch; ++b)
            for (int64_t h = 0; h < heads; ++h) {
                ExactGemm q2 = p;
                const int64_t bh = b * heads + h;
                q2.a = q + row_off(layout, b, h, heads, n, e);
                q2.b = k + row_off(layout, b, h, heads, n, e);
                q2.a_os = 0; q2.a_is = chunk * rs; q2.b_os = 0; q2.b_is = 0;
                q2.c = logits + bh * n * k_max; q2.c_os = 0; q2.c_is = chunk * k_max;
                q2.idx = idx + bh * nc * k_max; q2.counts = counts + bh * nc;
                cudaError_t err = launch_exact(q2, nc, s);
                if (err != cudaSuccess) return err;
            }
        return cudaSuccess;
    }
    // identity: full N x N logits per (b, h)
    p.M = n; p.N = n; p.K = e; p.inner = 1;
    p.ldc = n; p.c_is = 0; p.a_is = 0; p.b_is = 0;
    for (int64_t b = 0; b < batch; ++b)
        for (int64_t h = 0; h < heads; ++h) {
            ExactGemm q2 = p;
            const int64_t bh = b * heads + h;
            q2.a = q + row_off(layout, b, h, heads, n, e); q2.lda = rs;
            q2.b = k + row_off(layout, b, h, heads, n, e); q2.ldb = rs;
            q2.c = logits + bh * n * n;
            cudaError_t err = launch_exact(q2, 1, s);
            if (err != cudaSuccess) return err;
        }
    return cudaSuccess;
}

cudaError_t check_softmax(float* buf, int64_t rows, int64_t rows_per_batch, int64_t stride,
                          const int32_t* counts, int64_t full, float* row_max, float* exp_sum,
                          uint32_t* flags, cudaStream_t s) {
    const int threads = 128;
    k_softmax_rows<<<(unsigned)((rows + threads - 1) / threads), threads, 0, s>>>(
        buf, rows, rows_per_batch, stride, counts, full, row_max, exp_sum, flags);
    return cudaGetLastError();
}

cudaError_t check_attention_pv(const float* probs, const float* v, int layout, int64_t batch,
                               int64_t heads, int64_t n, int64_t e, int64_t chunk,
                               const int32_t* idx, const int32_t* counts, int64_t k_max,
                               const float* base, float scale, float* out, cudaStream_t s) {
    const int64_t rs = layout == CSD_LAYOUT_BHNE ? e : heads * e;
    ExactGemm p{};
    p.trans_b = false;
    p.N = e;
    p.ldc = rs;
    p.ldb = rs;
    if (idx) {
        const int64_t nc = n / chunk;
        p.M = chunk; p.K = k_max; p.lda = k_max;
        p.idx_stride = k_max; p.inner = nc;
        p.epi = 5; p.scale = scale;
        for (int64_t b = 0; b < batch; ++b)
            for (int64_t h = 0; h < heads; ++h) {
                ExactGemm q2 = p;
                const int64_t bh = b * heads + h;
                const int64_t off = row_off(layout, b, h, heads, n, e);
                q2.a = probs + bh * n * k_max; q2.a_os = 0; q2.a_is = chunk * k_max;
                q2.b = v + off; q2.b_os = 0; q2.b_is = 0;
                q2.c = out + off; q2.c_os = 0; q2.c_is = chunk * rs;
                q2.bias = base + off;
                q2.idx = idx + bh * nc * k_max; q2.counts = counts + bh * nc;
                cudaError_t err = launch_exact(q2, nc, s);
                if (err != cudaSuccess) return err;
            }
        return cudaSuccess;
    }
    p.M = n; p.K = n; p.lda = n; p.inner = 1; p.epi = 0;
    for (int64_t b = 0; b < batch; ++b)
        for (int64_t h = 0; h < heads; ++h) {
            ExactGemm q2 = p;
            const int64_t bh = b * heads + h;
            const int64_t off = row_off(layout, b, h, heads, n, e);
            q2.a = probs + bh * n * n;
            q2.b = v + off;
            q2.c = out + off;
            cudaError_t err = launch_exact(q2, 1, s);
            if (err != cudaSuccess) return err;
        }
    return cudaSuccess;
}

cudaError_t check_colsum(const float* logits, const float* m, const float* l, int64_t bh_count,
                         int64_t n, int64_t chunk, float* out, cudaStream_t s) {
    dim3 grid((unsigned)((n + 127) / 128), (unsigned)(n / chunk), (unsigned)bh_count);
    k_colsum_exact<<<grid, 128, 0, s>>>(logits, m, l, n, chunk, bh_count, out);
    return cudaGetLastError();
}

// x[B,N,D] @ w[D,Dout] per batch (model.cpp:107-120)
cudaError_t check_project(const float* x, const float* w, int64_t batch, int64_t n, int64_t d,
                          int64_t dout, float* out, cudaStream_t s) {
    ExactGemm p{};
    p.a = x; p.lda = d; p.b = w; p.ldb = dout; p.trans_b = false;
    p.c = out; p.ldc = dout; p.M = batch * n; p.N = dout; p.K = d; p.inner = 1; p.epi = 0;
    return launch_exact(p, 1, s);
}

cudaError_t check_add(const float* a, const float* b, int64_t numel, float* out, cudaStream_t s) {
    k_add_exact<<<(unsigned)((numel + 255) / 256), 256, 0, s>>>(a, b, numel, out);
    return cudaGetLastError();
}

// dense_mlp (mlp.cpp:49-81): act = gelu(x W1^T + b1) into act_ref [B,N,F];
// out = act W2 + b2.
cudaError_t check_dense_mlp(const float* x, const float* w1, const float* b1, const float* w2,
                            const float* b2, int64_t batch, int64_t n, int64_t d, int64_t f,
                            float* act_ref, float* out, cudaStream_t s) {
    ExactGemm p{};
    p.a = x; p.lda = d; p.b = w1; p.ldb = d; p.trans_b = true;
    p.c = act_ref; p.ldc = f; p.M = batch * n; p.N = f; p.K = d; p.inner = 1;
    p.epi = 3; p.bias = b1;
    cudaError_t err = launch_exact(p, 1, s);
    if (err != cudaSuccess) return err;
    ExactGemm q{};
    q.a = act_ref; q.lda = f; q.b = w2; q.ldb = d; q.trans_b = false;
    q.c = out; q.ldc = d; q.M = batch * n; q.N = d; q.K = f; q.inner = 1;
    q.epi = 2; q.bias = b2;
    return launch_exact(q, 1, s);
}

// mlp_tile_means (mlp.cpp:83-96) into out [B, C, F]; means_ws [B*C, D].
cudaError_t check_tile_means(const float* x, const float* w1, int64_t batch, int64_t n, int64_t d,
                             int64_t f, int64_t chunk, float* means_ws, float* out,
                             cudaStream_t s) {
    const int64_t nc = n / chunk;
    dim3 grid((unsigned)((d + 127) / 128), (unsigned)(batch * nc));
    k_chunk_mean_exact<<<grid, 128, 0, s>>>(x, batch, n, d, chunk, means_ws);
    ExactGemm p{};
    p.a = means_ws; p.lda = d; p.b = w1; p.ldb = d; p.trans_b = true;
    p.c = out; p.ldc = f; p.M = batch * nc; p.N = f; p.K = d; p.inner = 1; p.epi = 0;
    return launch_exact(p, 1, s);
}

cudaError_t check_absdiff(const float* a, const float* b, int64_t numel, float* out,
                          cudaStream_t s) {
    k_absdiff<<<(unsigned)((numel + 255) / 256), 256, 0, s>>>(a, b, numel, out);
    return cudaGetLastError();
}

// sparse_delta_mlp (mlp.cpp:120-182).  ws: [B*C*chunk, k_max] pre/delta.
cudaError_t check_sparse_delta_mlp(const float* x, const float* w1, const float* b1,
                                   const float* w2, const int32_t* idx, const int32_t* counts,
                                   int64_t k_max, int64_t chunk, int64_t batch, int64_t n,
                                   int64_t d, int64_t f, float* act_ref, float* out_cache,
                                   float* ws, cudaStream_t s) {
    const int64_t nc = n / chunk;
    const int64_t total = batch * nc;
    ExactGemm p{};
    p.a = x; p.lda = d; p.a_os = chunk * d; p.a_is = 0;
    p.b = w1; p.ldb = d; p.trans_b = true;
    p.c = ws; p.ldc = k_max; p.c_os = chunk * k_max; p.c_is = 0;
    p.M = chunk; p.N = k_max; p.K = d; p.inner = 1;
    p.idx = idx; p.counts = counts; p.idx_stride = k_max;
    p.epi = 3; p.bias = b1;
    cudaError_t err = launch_exact(p, total, s);
    if (err != cudaSuccess) return err;
    dim3 g2((unsigned)((k_max + 127) / 128), (unsigned)(total * chunk));
    k_mlp_refresh_exact<<<g2, 128, 0, s>>>(ws, idx, counts, k_max, chunk, n, f, total, act_ref);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    ExactGemm q{};
    q.a = ws; q.lda = k_max; q.a_os = chunk * k_max; q.a_is = 0;
    q.b = w2; q.ldb = d; q.trans_b = false;
    q.c = out_cache; q.ldc = d; q.c_os = chunk * d; q.c_is = 0;
    q.M = chunk; q.N = d; q.K = k_max; q.inner = 1;
    q.idx = idx; q.counts = counts; q.idx_stride = k_max;
    q.epi = 4;
    return launch_exact(q, total, s);
}

}  // namespace dev
}  // namespace csd

namespace csd {
namespace dev {
// pre = x W1^T + b1 (mlp.cpp:55-59), the MlpDenseResult::preact view.
cudaError_t check_mlp_preact(const float* x, const float* w1, const float* b1, int64_t rows,
                             int64_t d, int64_t f, float* pre, cudaStream_t s) {
    ExactGemm p{};
    p.a = x; p.lda = d; p.b = w1; p.ldb = d; p.trans_b = true;
    p.c = pre; p.ldc = f; p.M = rows; p.N = f; p.K = d; p.inner = 1;
    p.epi = 2; p.bias = b1;
    return launch_exact(p, 1, s);
}
}  // namespace dev
}  // namespace csd
