/*
 * csd_oracle.c — TEST INFRASTRUCTURE ONLY (see csd_oracle.h).
 *
 * CPU restatement of the reference's hot path, written in plain C.  Every
 * function cites the reference routine it restates; the arithmetic order is
 * kept op-for-op so the result is bit-identical to the reference build
 * (g++ -O3, x86-64 baseline: no FMA contraction, glibc expf/tanhf).
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (oracle/Makefile).
 * Pinned against: the compiled reference (oracle/_ref, tests/golden/*.npz
 * made by oracle/gen_golden.py) and the reference's own known-answer tests
 * (tests/test_oracle.py).
 */
#include "csd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* glibc 2.39 expf (sysdeps/ieee754/flt-32/e_expf.c, EXP2F_TABLE_BITS = 5). */
/* Table entries: bits(2^(i/32)) - (i << 47), regenerated from first
 * principles by oracle/gen_exp2_table.py.  The x86-64 FMA ifunc variant
 * contracts `r = z - kd` into fma(InvLn2N, xd, -kd); with that contraction
 * this restatement agrees with the host libm on all 2,240,806,912 finite
 * floats in (-110, 90) (exhaustive sweep, oracle/check_expf_exhaustive.c). */
static const uint64_t kExp2Tab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull,
};

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static inline uint64_t d2u(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static inline double u2d(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }

float csdo_expf(float x) {
    const double inv_ln2_n = 0x1.71547652b82fep+0 * 32;
    const double shift = 0x1.8p+52;
    const double c0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32;
    const double c1 = 0x1.ebfce50fac4f3p-3 / 32 / 32;
    const double c2 = 0x1.62e42ff0c52d6p-1 / 32;
    const uint32_t abstop = (f2u(x) >> 20) & 0x7ff;
    if (abstop >= (f2u(88.0f) >> 20)) {
        if (f2u(x) == f2u(-INFINITY)) return 0.0f;
        if (abstop >= (f2u(INFINITY) >> 20)) return x + x;
        if (x > 0x1.62e42ep6f) return INFINITY;
        if (x < -0x1.9fe368p6f) return 0.0f;
    }
    const double xd = (double)x;
    const double z = inv_ln2_n * xd;
    double kd = z + shift;
    const uint64_t ki = d2u(kd);
    kd -= shift;
    const double r = fma(inv_ln2_n, xd, -kd);
    uint64_t t = kExp2Tab[ki % 32];
    t += ki << 47;
    const double s = u2d(t);
    const double p = c0 * r + c1;
    const double r2 = r * r;
    double y = c2 * r + 1.0;
    y = p * r2 + y;
    y = y * s;
    return (float)y;
}

/* glibc 2.39 expm1f / tanhf (fdlibm s_expm1f.c with the 5-term Q polynomial,
 * s_tanhf.c).  Agrees with the host libm tanhf on every non-NaN float
 * (exhaustive sweep of all 2^32 patterns, oracle/check_tanhf_exhaustive.c). */
static float csdo_expm1f(float x) {
    const float one = 1.0f, huge = 1.0e+30f, tiny = 1.0e-30f;
    const float o_threshold = 8.8721679688e+01f, ln2_hi = 6.9313812256e-01f,
                ln2_lo = 9.0580006145e-06f, invln2 = 1.4426950216e+00f;
    const float q1 = -3.3333335072e-02f, q2 = 1.5873016091e-03f, q3 = -7.9365076090e-05f,
                q4 = 4.0082177293e-06f, q5 = -2.0109921195e-07f;
    float y, hi, lo, c = 0.0f, t, e, hxs, hfx, r1;
    int32_t k;
    uint32_t hx = f2u(x);
    const uint32_t xsb = hx & 0x80000000u;
    hx &= 0x7fffffffu;
    if (hx >= 0x4195b844u) {
        if (hx >= 0x42b17218u) {
            if (hx > 0x7f800000u) return x + x;
            if (hx == 0x7f800000u) return (xsb == 0) ? x : -1.0f;
            if (x > o_threshold) return huge * huge;
        }
        if (xsb != 0) return tiny - one;
    }
    if (hx > 0x3eb17218u) {
        if (hx < 0x3F851592u) {
            if (xsb == 0) { hi = x - ln2_hi; lo = ln2_lo; k = 1; }
            else { hi = x + ln2_hi; lo = -ln2_lo; k = -1; }
        } else {
            k = (int32_t)(invln2 * x + ((xsb == 0) ? 0.5f : -0.5f));
            t = (float)k;
            hi = x - t * ln2_hi;
            lo = t * ln2_lo;
        }
        x = hi - lo;
        c = (hi - x) - lo;
    } else if (hx < 0x33000000u) {
        t = huge + x;
        return x - (t - (huge + x));
    } else {
        k = 0;
    }
    hfx = 0.5f * x;
    hxs = x * hfx;
    r1 = one + hxs * (q1 + hxs * (q2 + hxs * (q3 + hxs * (q4 + hxs * q5))));
    t = 3.0f - r1 * hfx;
    e = hxs * ((r1 - t) / (6.0f - x * t));
    if (k == 0) return x - (x * e - hxs);
    e = (x * (e - c) - c);
    e -= hxs;
    if (k == -1) return 0.5f * (x - e) - 0.5f;
    if (k == 1) {
        if (x < -0.25f) return -2.0f * (e - (x + 0.5f));
        return one + 2.0f * (x - e);
    }
    if (k <= -2 || k > 56) {
        y = one - (e - x);
        y = u2f(f2u(y) + ((uint32_t)k << 23));
        return y - one;
    }
    if (k < 23) {
        t = u2f(0x3f800000u - (0x1000000u >> k));
        y = t - (e - x);
        y = u2f(f2u(y) + ((uint32_t)k << 23));
    } else {
        t = u2f((uint32_t)(0x7f - k) << 23);
        y = x - (e + t);
        y += one;
        y = u2f(f2u(y) + ((uint32_t)k << 23));
    }
    return y;
}

float csdo_tanhf(float x) {
    const float one = 1.0f, two = 2.0f, tiny = 1.0e-30f;
    float t, z;
    const int32_t jx = (int32_t)f2u(x);
    const int32_t ix = jx & 0x7fffffff;
    if (ix >= 0x7f800000) return (jx >= 0) ? one / x + one : one / x - one;
    if (ix < 0x41b00000) {
        if (ix == 0) return x;
        if (ix < 0x24000000) return x * (one + x);
        if (ix >= 0x3f800000) {
            t = csdo_expm1f(two * fabsf(x));
            z = one - two / (t + two);
        } else {
            t = csdo_expm1f(-two * fabsf(x));
            z = -t / (t + two);
        }
    } else {
        z = one - tiny;
    }
    return (jx >= 0) ? z : -z;
}

/* tensor.cpp:141-152: 0.5*v*(1 + tanh(sqrt(2/pi)*(v + 0.044715*v^3))). */
float csdo_gelu(float v) {
    const float k = sqrtf(2.0f / (float)M_PI);
    const float cube = 0.044715f * v * v * v;
    return 0.5f * v * (1.0f + csdo_tanhf(k * (v + cube)));
}

/* ------------------------------------------------------------------------ */
/* voxel.cpp:7-42 */
int csdo_voxel_permutation(int64_t t, int64_t h, int64_t w, int64_t vt, int64_t vh, int64_t vw,
                           int64_t* perm) {
    if (t < 1 || h < 1 || w < 1 || vt < 1 || vh < 1 || vw < 1) return CSDO_ECONFIG;
    if (t % vt || h % vh || w % vw) return CSDO_ECONFIG;
    int64_t pos = 0;
    for (int64_t tc = 0; tc < t / vt; ++tc)
        for (int64_t hc = 0; hc < h / vh; ++hc)
            for (int64_t wc = 0; wc < w / vw; ++wc)
                for (int64_t it = 0; it < vt; ++it)
                    for (int64_t ih = 0; ih < vh; ++ih)
                        for (int64_t iw = 0; iw < vw; ++iw)
                            perm[pos++] = ((tc * vt + it) * h + hc * vh + ih) * w + wc * vw + iw;
    return CSDO_OK;
}

static int voxel_move(const float* x, int64_t batch, int64_t t, int64_t h, int64_t w, int64_t d,
                      int64_t vt, int64_t vh, int64_t vw, float* out, int scatter) {
    const int64_t n = t * h * w;
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    const int rc = csdo_voxel_permutation(t, h, w, vt, vh, vw, perm);
    if (rc) { free(perm); return rc; }
    for (int64_t b = 0; b < batch; ++b) {
        const float* src = x + b * n * d;
        float* dst = out + b * n * d;
        for (int64_t pos = 0; pos < n; ++pos) {
            if (scatter) memcpy(dst + perm[pos] * d, src + pos * d, sizeof(float) * (size_t)d);
            else memcpy(dst + pos * d, src + perm[pos] * d, sizeof(float) * (size_t)d);
        }
    }
    free(perm);
    return CSDO_OK;
}

/* voxel.cpp:44-73 */
int csdo_voxel_order(const float* x, int64_t batch, int64_t t, int64_t h, int64_t w, int64_t d,
                     int64_t vt, int64_t vh, int64_t vw, float* out) {
    return voxel_move(x, batch, t, h, w, d, vt, vh, vw, out, 0);
}

/* voxel.cpp:75-102 */
int csdo_reverse_voxel_order(const float* x, int64_t batch, int64_t t, int64_t h, int64_t w,
                             int64_t d, int64_t vt, int64_t vh, int64_t vw, float* out) {
    return voxel_move(x, batch, t, h, w, d, vt, vh, vw, out, 1);
}

/* ------------------------------------------------------------------------ */
/* sparse_index.cpp:64-96.  The comparator (s[a] != s[b] ? s[a] > s[b] : a < b)
 * is a strict total order on non-NaN rows, so the selected prefix is unique;
 * we select it with a bounded min-heap on the same order.                  */
static const float* g_row;
static int before(int32_t a, int32_t b) { /* true if a ranks ahead of b */
    if (g_row[a] != g_row[b]) return g_row[a] > g_row[b];
    return a < b;
}
static void sift_down(int32_t* heap, int64_t size, int64_t i) {
    /* heap root = worst-ranked kept element */
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < size && before(heap[m], heap[l])) m = l;
        if (r < size && before(heap[m], heap[r])) m = r;
        if (m == i) return;
        int32_t tmp = heap[i]; heap[i] = heap[m]; heap[m] = tmp;
        i = m;
    }
}
int csdo_select_top_k(const float* scores, int64_t rows, int64_t m, int64_t k, int32_t* idx_out) {
    if (k < 1 || k > m) return CSDO_EVALUE;
    int32_t* heap = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
    for (int64_t r = 0; r < rows; ++r) {
        g_row = scores + r * m;
        for (int64_t j = 0; j < k; ++j) heap[j] = (int32_t)j;
        for (int64_t i = k / 2 - 1; i >= 0; --i) sift_down(heap, k, i);
        for (int64_t j = k; j < m; ++j) {
            if (before((int32_t)j, heap[0])) { heap[0] = (int32_t)j; sift_down(heap, k, 0); }
        }
        /* pop worst-first into descending-rank order */
        int32_t* dst = idx_out + r * k;
        for (int64_t s = k; s > 0; --s) {
            dst[s - 1] = heap[0];
            heap[0] = heap[s - 1];
            sift_down(heap, s - 1, 0);
        }
    }
    free(heap);
    return CSDO_OK;
}

/* sparse_index.cpp:27-62 */
int csdo_validate_index_set(const int32_t* idx, const int32_t* counts, int64_t rows, int64_t k_max,
                            int64_t domain) {
    if (k_max < 0 || k_max > domain) return CSDO_EVALUE;
    unsigned char* seen = (unsigned char*)calloc((size_t)domain, 1);
    int rc = CSDO_OK;
    for (int64_t r = 0; r < rows && rc == CSDO_OK; ++r) {
        const int32_t cnt = counts[r];
        if (cnt < 0 || cnt > k_max) { rc = CSDO_EVALUE; break; }
        const int32_t* ids = idx + r * k_max;
        for (int32_t j = 0; j < cnt; ++j) {
            if (ids[j] < 0 || ids[j] >= domain) { rc = CSDO_EINDEX; break; }
            if (seen[ids[j]]) { rc = CSDO_EINDEX; break; }
            seen[ids[j]] = 1;
        }
        for (int32_t j = 0; j < cnt; ++j)
            if (ids[j] >= 0 && ids[j] < domain) seen[ids[j]] = 0;
    }
    free(seen);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* tensor.cpp:66-98: acc starts at 0, `acc += a*b` in k order. */
void csdo_gemm(const float* a, const float* b, int64_t m, int64_t kk, int64_t n, int transpose_b,
               float* out) {
    for (int64_t i = 0; i < m; ++i) {
        const float* ra = a + i * kk;
        for (int64_t j = 0; j < n; ++j) {
            float acc = 0.0f;
            if (transpose_b) {
                const float* rb = b + j * kk;
                for (int64_t k = 0; k < kk; ++k) acc += ra[k] * rb[k];
            } else {
                for (int64_t k = 0; k < kk; ++k) acc += ra[k] * b[k * n + j];
            }
            out[i * n + j] = acc;
        }
    }
}

/* tensor.cpp:100-139 */
int csdo_softmax_rows(const float* logits, int64_t rows, int64_t len, float* probs, float* row_max,
                      float* exp_sum) {
    for (int64_t r = 0; r < rows; ++r) {
        const float* row = logits + r * len;
        float m = row[0];
        for (int64_t j = 0; j < len; ++j) {
            if (!isfinite(row[j])) return CSDO_ENUMERIC;
            if (row[j] > m) m = row[j];
        }
        float l = 0.0f;
        float* o = probs + r * len;
        for (int64_t j = 0; j < len; ++j) {
            o[j] = csdo_expf(row[j] - m);
            l += o[j];
        }
        for (int64_t j = 0; j < len; ++j) o[j] /= l;
        if (row_max) row_max[r] = m;
        if (exp_sum) exp_sum[r] = l;
    }
    return CSDO_OK;
}

/* attention.cpp:38-44 */
static void scaled_logits(const float* q, const float* k, int64_t rows, int64_t n, int64_t e,
                          float* out) {
    csdo_gemm(q, k, rows, e, n, 1, out);
    const float scale = 1.0f / sqrtf((float)e);
    for (int64_t i = 0; i < rows * n; ++i) out[i] *= scale;
}

/* attention.cpp:59-74 */
int csdo_dense_attention(const float* q, const float* k, const float* v, int64_t batch,
                         int64_t heads, int64_t n, int64_t e, float* out) {
    float* logits = (float*)malloc(sizeof(float) * (size_t)(n * n));
    float* probs = (float*)malloc(sizeof(float) * (size_t)(n * n));
    int rc = CSDO_OK;
    for (int64_t bh = 0; bh < batch * heads && rc == CSDO_OK; ++bh) {
        const int64_t off = bh * n * e;
        scaled_logits(q + off, k + off, n, n, e, logits);
        rc = csdo_softmax_rows(logits, n, n, probs, NULL, NULL);
        if (rc == CSDO_OK) csdo_gemm(probs, v + off, n, n, e, 0, out + off);
    }
    free(logits);
    free(probs);
    return rc;
}

/* attention.cpp:76-145 */
int csdo_column_sum_attention(const float* q, const float* k, const float* v, const float* prev_m,
                              const float* prev_l, int64_t batch, int64_t heads, int64_t n,
                              int64_t e, int64_t chunk, float* out, float* row_max,
                              float* exp_sum, float* column_sums) {
    if (chunk < 1 || n % chunk) return CSDO_ESHAPE;
    float* logits = (float*)malloc(sizeof(float) * (size_t)(n * n));
    float* probs = (float*)malloc(sizeof(float) * (size_t)(n * n));
    int rc = CSDO_OK;
    const int64_t nc = n / chunk;
    for (int64_t bh = 0; bh < batch * heads && rc == CSDO_OK; ++bh) {
        const int64_t off = bh * n * e;
        scaled_logits(q + off, k + off, n, n, e, logits);
        rc = csdo_softmax_rows(logits, n, n, probs, row_max + bh * n, exp_sum + bh * n);
        if (rc) break;
        csdo_gemm(probs, v + off, n, n, e, 0, out + off);
        const float* um = prev_m ? prev_m + bh * n : row_max + bh * n;
        const float* ul = prev_l ? prev_l + bh * n : exp_sum + bh * n;
        /* p_approx = exp(logit - m)/l (:131-137), then chunk_reduce Sum (:138,
         * tensor.cpp:188-225: w = 0; w += row, rows in order). */
        float* cs = column_sums + bh * nc * n;
        for (int64_t c = 0; c < nc; ++c) {
            float* w = cs + c * n;
            for (int64_t j = 0; j < n; ++j) w[j] = 0.0f;
            for (int64_t i = c * chunk; i < (c + 1) * chunk; ++i) {
                const float m = um[i], l = ul[i];
                for (int64_t j = 0; j < n; ++j) w[j] += csdo_expf(logits[i * n + j] - m) / l;
            }
        }
    }
    free(logits);
    free(probs);
    return rc;
}

/* attention.cpp:147-194 */
int csdo_sparse_delta_attention(const float* q, const float* k, const float* v,
                                const int32_t* idx, const int32_t* counts, int64_t k_max,
                                int64_t chunk, const float* base, float scale, int64_t batch,
                                int64_t heads, int64_t n, int64_t e, float* out) {
    if (chunk < 1 || n % chunk) return CSDO_ESHAPE;
    const int64_t nc = n / chunk;
    int rc = csdo_validate_index_set(idx, counts, batch * heads * nc, k_max, n);
    if (rc) return rc;
    if (out != base) memcpy(out, base, sizeof(float) * (size_t)(batch * heads * n * e));
    float* ksel = (float*)malloc(sizeof(float) * (size_t)((k_max ? k_max : 1) * e));
    float* vsel = (float*)malloc(sizeof(float) * (size_t)((k_max ? k_max : 1) * e));
    float* logits = (float*)malloc(sizeof(float) * (size_t)(chunk * (k_max ? k_max : 1)));
    float* probs = (float*)malloc(sizeof(float) * (size_t)(chunk * (k_max ? k_max : 1)));
    float* delta = (float*)malloc(sizeof(float) * (size_t)(chunk * e));
    const float inv_sqrt_e = 1.0f / sqrtf((float)e);
    for (int64_t bh = 0; bh < batch * heads && rc == CSDO_OK; ++bh) {
        const int64_t off = bh * n * e;
        for (int64_t c = 0; c < nc; ++c) {
            const int32_t cnt = counts[bh * nc + c];
            if (cnt == 0) continue;
            const int32_t* ids = idx + (bh * nc + c) * k_max;
            for (int32_t j = 0; j < cnt; ++j) {
                memcpy(ksel + j * e, k + off + (int64_t)ids[j] * e, sizeof(float) * (size_t)e);
                memcpy(vsel + j * e, v + off + (int64_t)ids[j] * e, sizeof(float) * (size_t)e);
            }
            csdo_gemm(q + off + c * chunk * e, ksel, chunk, e, cnt, 1, logits);
            for (int64_t i = 0; i < chunk * cnt; ++i) logits[i] *= inv_sqrt_e;
            rc = csdo_softmax_rows(logits, chunk, cnt, probs, NULL, NULL);
            if (rc) break;
            csdo_gemm(probs, vsel, chunk, cnt, e, 0, delta);
            float* dst = out + off + c * chunk * e;
            for (int64_t i = 0; i < chunk * e; ++i) dst[i] += scale * delta[i];
        }
    }
    free(ksel); free(vsel); free(logits); free(probs); free(delta);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* mlp.cpp:49-81 */
int csdo_dense_mlp(const float* x, const float* w1, const float* b1, const float* w2,
                   const float* b2, int64_t batch, int64_t n, int64_t d, int64_t f, float* out,
                   float* pre_out, float* act_out) {
    float* pre = (float*)malloc(sizeof(float) * (size_t)(n * f));
    float* act = (float*)malloc(sizeof(float) * (size_t)(n * f));
    for (int64_t b = 0; b < batch; ++b) {
        csdo_gemm(x + b * n * d, w1, n, d, f, 1, pre);
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < f; ++j) pre[i * f + j] += b1[j];
        for (int64_t i = 0; i < n * f; ++i) act[i] = csdo_gelu(pre[i]);
        float* o = out + b * n * d;
        csdo_gemm(act, w2, n, f, d, 0, o);
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < d; ++j) o[i * d + j] += b2[j];
        if (pre_out) memcpy(pre_out + b * n * f, pre, sizeof(float) * (size_t)(n * f));
        if (act_out) memcpy(act_out + b * n * f, act, sizeof(float) * (size_t)(n * f));
    }
    free(pre);
    free(act);
    return CSDO_OK;
}

/* mlp.cpp:83-96 with chunk_reduce Mean (tensor.cpp:188-225). */
int csdo_mlp_tile_means(const float* x, const float* w1, int64_t batch, int64_t n, int64_t d,
                        int64_t f, int64_t chunk, float* out) {
    if (chunk < 1 || n % chunk) return CSDO_ESHAPE;
    const int64_t nc = n / chunk;
    const float inv = 1.0f / (float)chunk;
    float* means = (float*)malloc(sizeof(float) * (size_t)(nc * d));
    for (int64_t b = 0; b < batch; ++b) {
        for (int64_t c = 0; c < nc; ++c) {
            float* w = means + c * d;
            for (int64_t j = 0; j < d; ++j) w[j] = 0.0f;
            for (int64_t r = c * chunk; r < (c + 1) * chunk; ++r)
                for (int64_t j = 0; j < d; ++j) w[j] += x[(b * n + r) * d + j];
            for (int64_t j = 0; j < d; ++j) w[j] *= inv;
        }
        csdo_gemm(means, w1, nc, d, f, 1, out + b * nc * f);
    }
    free(means);
    return CSDO_OK;
}

/* mlp.cpp:98-118 */
int csdo_mlp_change_indices(const float* x, const float* w1, const float* tile_means,
                            int64_t batch, int64_t n, int64_t d, int64_t f, int64_t k,
                            int64_t chunk, int32_t* idx_out) {
    if (chunk < 1 || n % chunk) return CSDO_ESHAPE;
    if (k < 1 || k > f) return CSDO_EVALUE;
    const int64_t nc = n / chunk;
    float* fresh = (float*)malloc(sizeof(float) * (size_t)(batch * nc * f));
    csdo_mlp_tile_means(x, w1, batch, n, d, f, chunk, fresh);
    for (int64_t i = 0; i < batch * nc * f; ++i) fresh[i] = fabsf(fresh[i] - tile_means[i]);
    const int rc = csdo_select_top_k(fresh, batch * nc, f, k, idx_out);
    free(fresh);
    return rc;
}

/* mlp.cpp:120-182 */
int csdo_sparse_delta_mlp(const float* x, const float* w1, const float* b1, const float* w2,
                          const int32_t* idx, const int32_t* counts, int64_t k_max,
                          int64_t chunk, int64_t batch, int64_t n, int64_t d, int64_t f,
                          float* act_cache, float* out_cache) {
    if (chunk < 1 || n % chunk) return CSDO_ESHAPE;
    const int64_t nc = n / chunk;
    int rc = csdo_validate_index_set(idx, counts, batch * nc, k_max, f);
    if (rc) return rc;
    const int64_t kk = k_max ? k_max : 1;
    float* w1s = (float*)malloc(sizeof(float) * (size_t)(kk * d));
    float* w2s = (float*)malloc(sizeof(float) * (size_t)(kk * d));
    float* pre = (float*)malloc(sizeof(float) * (size_t)(chunk * kk));
    float* dl = (float*)malloc(sizeof(float) * (size_t)(chunk * kk));
    float* contrib = (float*)malloc(sizeof(float) * (size_t)(chunk * d));
    for (int64_t b = 0; b < batch; ++b) {
        for (int64_t c = 0; c < nc; ++c) {
            const int32_t cnt = counts[b * nc + c];
            if (cnt == 0) continue;
            const int32_t* ids = idx + (b * nc + c) * k_max;
            for (int32_t j = 0; j < cnt; ++j) {
                memcpy(w1s + j * d, w1 + (int64_t)ids[j] * d, sizeof(float) * (size_t)d);
                memcpy(w2s + j * d, w2 + (int64_t)ids[j] * d, sizeof(float) * (size_t)d);
            }
            const float* xc = x + (b * n + c * chunk) * d;
            csdo_gemm(xc, w1s, chunk, d, cnt, 1, pre);
            for (int64_t r = 0; r < chunk; ++r)
                for (int32_t j = 0; j < cnt; ++j) pre[r * cnt + j] += b1[ids[j]];
            float* ac = act_cache + (b * n + c * chunk) * f;
            for (int64_t r = 0; r < chunk; ++r) {
                for (int32_t j = 0; j < cnt; ++j) {
                    const float fresh = csdo_gelu(pre[r * cnt + j]);
                    float* cached = ac + r * f + ids[j];
                    dl[r * cnt + j] = fresh - *cached;
                    *cached = fresh;
                }
            }
            csdo_gemm(dl, w2s, chunk, cnt, d, 0, contrib);
            float* dst = out_cache + (b * n + c * chunk) * d;
            for (int64_t i = 0; i < chunk * d; ++i) dst[i] += contrib[i];
        }
    }
    free(w1s); free(w2s); free(pre); free(dl); free(contrib);
    return CSDO_OK;
}

/* ------------------------------------------------------------------------ */
/* model.cpp:107-120 */
void csdo_project(const float* x, const float* w, int64_t batch, int64_t n, int64_t d,
                  int64_t dout, float* out) {
    for (int64_t b = 0; b < batch; ++b) csdo_gemm(x + b * n * d, w, n, d, dout, 0, out + b * n * dout);
}

/* model.cpp:122-142 */
void csdo_split_heads(const float* x, int64_t batch, int64_t n, int64_t heads, int64_t e,
                      float* out) {
    for (int64_t b = 0; b < batch; ++b)
        for (int64_t t = 0; t < n; ++t)
            for (int64_t h = 0; h < heads; ++h)
                memcpy(out + ((b * heads + h) * n + t) * e, x + ((b * n + t) * heads + h) * e,
                       sizeof(float) * (size_t)e);
}

/* model.cpp:144-165 */
void csdo_merge_heads(const float* x, int64_t batch, int64_t heads, int64_t n, int64_t e,
                      float* out) {
    for (int64_t b = 0; b < batch; ++b)
        for (int64_t h = 0; h < heads; ++h)
            for (int64_t t = 0; t < n; ++t)
                memcpy(out + ((b * n + t) * heads + h) * e, x + ((b * heads + h) * n + t) * e,
                       sizeof(float) * (size_t)e);
}

/* ------------------------------------------------------------------------ */
/* rng.hpp:12-44 (GaussianRng: std::mt19937_64 + Box-Muller, spare cached) as
 * used by tests/test_util.hpp:50-55 random_tensor and model.cpp:32-37.      */
typedef struct { uint64_t mt[312]; int idx; } mt64_t;
static void mt64_seed(mt64_t* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}
static uint64_t mt64_next(mt64_t* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t y = (g->mt[i] & 0xFFFFFFFF80000000ull) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFull);
            g->mt[i] = g->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ull : 0);
        }
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}
void csdo_gaussian(uint64_t seed, int64_t n, float stddev, float* out) {
    mt64_t* g = (mt64_t*)malloc(sizeof(mt64_t));
    mt64_seed(g, seed);
    int have_spare = 0;
    float spare = 0.0f;
    for (int64_t i = 0; i < n; ++i) {
        if (have_spare) {
            have_spare = 0;
            out[i] = 0.0f + stddev * spare;
            continue;
        }
        double u1;
        do { u1 = (double)(mt64_next(g) >> 11) * (1.0 / 9007199254740992.0); } while (u1 <= 1e-300);
        const double u2 = (double)(mt64_next(g) >> 11) * (1.0 / 9007199254740992.0);
        const double r = sqrt(-2.0 * log(u1));
        const double theta = 2.0 * M_PI * u2;
        spare = (float)(r * sin(theta));
        have_spare = 1;
        out[i] = 0.0f + stddev * (float)(r * cos(theta));
    }
    free(g);
}

/* ------------------------------------------------------------------------ */
/* Self-check hook for tests/test_oracle.py: number of float bit patterns in
 * [start, stop) (stride `step`) where csdo_expf / csdo_tanhf differ from the
 * host libm's expf / tanhf.  NaN patterns are skipped.                      */
int64_t csdo_libm_mismatches(uint32_t start, uint32_t stop, uint32_t step, int which) {
    int64_t bad = 0;
    for (uint64_t u = start; u < stop; u += step) {
        const float x = u2f((uint32_t)u);
        if (isnan(x)) continue;
        const float a = which == 0 ? csdo_expf(x) : csdo_tanhf(x);
        const float b = which == 0 ? expf(x) : tanhf(x);
        if (f2u(a) != f2u(b)) ++bad;
    }
    return bad;
}
