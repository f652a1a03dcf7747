// common.cuh — shared device helpers for the csd_b200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "csd_b200.h"
#include "kernels.h"

namespace csd {
namespace dev {

__device__ __forceinline__ void raise_flag(uint32_t* flags, uint32_t bit) {
    if (flags) atomicOr(flags, bit);
}

// Programmatic dependent launch (launch_util.h launch_ex): a kernel launched behind another
// one of the block step may start its prologue (barrier init, TMEM allocation, code warm-up)
// while the previous kernel drains.  pdl_wait() -- before the first global-memory access --
// blocks until the previous grid has completed and its writes are visible (a no-op for a
// plain launch); pdl_trigger() lets the NEXT kernel's CTAs be scheduled once every CTA of
// this grid has triggered or exited.  Called after pdl_wait(), so a kernel's prologue only
// ever overlaps its direct predecessor.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Exact (reference-reproducing) scalar math for CSD_MODE_CHECK.
//
// glibc 2.39 expf restated in IEEE double with explicit rounding intrinsics
// so nvcc cannot contract or reassociate; identical op sequence to
// oracle/csd_oracle.c:csdo_expf (pinned there against host libm over every
// float in (-110, 90)).
static __constant__ uint64_t kExp2Tab32[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull,
};

__device__ __forceinline__ float exact_expf(float x) {
    const double inv_ln2_n = 0x1.71547652b82fep+0 * 32;
    const double shift = 0x1.8p+52;
    const double c0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32;
    const double c1 = 0x1.ebfce50fac4f3p-3 / 32 / 32;
    const double c2 = 0x1.62e42ff0c52d6p-1 / 32;
    const uint32_t ux = __float_as_uint(x);
    const uint32_t abstop = (ux >> 20) & 0x7ff;
    if (abstop >= (0x42b00000u >> 20)) {            // |x| >= 88 or non-finite
        if (ux == 0xff800000u) return 0.0f;         // -inf
        if (abstop >= (0x7f800000u >> 20)) return __fadd_rn(x, x);
        if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);
        if (x < -0x1.9fe368p6f) return 0.0f;
    }
    const double xd = (double)x;
    const double z = __dmul_rn(inv_ln2_n, xd);
    double kd = __dadd_rn(z, shift);
    const uint64_t ki = (uint64_t)__double_as_longlong(kd);
    kd = __dsub_rn(kd, shift);
    const double r = __fma_rn(inv_ln2_n, xd, -kd);
    uint64_t t = kExp2Tab32[ki % 32];
    t += ki << 47;
    const double s = __longlong_as_double((long long)t);
    const double p = __dadd_rn(__dmul_rn(c0, r), c1);
    const double r2 = __dmul_rn(r, r);
    double y = __dadd_rn(__dmul_rn(c2, r), 1.0);
    y = __dadd_rn(__dmul_rn(p, r2), y);
    y = __dmul_rn(y, s);
    return __double2float_rn(y);
}

// glibc 2.39 expm1f / tanhf (fdlibm), float ops with explicit rounding.
__device__ __forceinline__ float exact_expm1f(float x) {
    const float one = 1.0f, huge = 1.0e+30f, tiny = 1.0e-30f;
    const float o_threshold = 8.8721679688e+01f, ln2_hi = 6.9313812256e-01f,
                ln2_lo = 9.0580006145e-06f, invln2 = 1.4426950216e+00f;
    const float q1 = -3.3333335072e-02f, q2 = 1.5873016091e-03f, q3 = -7.9365076090e-05f,
                q4 = 4.0082177293e-06f, q5 = -2.0109921195e-07f;
    float y, hi, lo, c = 0.0f, t, e, hxs, hfx, r1;
    int32_t k;
    uint32_t hx = __float_as_uint(x);
    const uint32_t xsb = hx & 0x80000000u;
    hx &= 0x7fffffffu;
    if (hx >= 0x4195b844u) {
        if (hx >= 0x42b17218u) {
            if (hx > 0x7f800000u) return __fadd_rn(x, x);
            if (hx == 0x7f800000u) return (xsb == 0) ? x : -1.0f;
            if (x > o_threshold) return __fmul_rn(huge, huge);
        }
        if (xsb != 0) return __fsub_rn(tiny, one);
    }
    if (hx > 0x3eb17218u) {
        if (hx < 0x3F851592u) {
            if (xsb == 0) { hi = __fsub_rn(x, ln2_hi); lo = ln2_lo; k = 1; }
            else { hi = __fadd_rn(x, ln2_hi); lo = -ln2_lo; k = -1; }
        } else {
            k = __float2int_rz(__fadd_rn(__fmul_rn(invln2, x), (xsb == 0) ? 0.5f : -0.5f));
            t = (float)k;
            hi = __fsub_rn(x, __fmul_rn(t, ln2_hi));
            lo = __fmul_rn(t, ln2_lo);
        }
        x = __fsub_rn(hi, lo);
        c = __fsub_rn(__fsub_rn(hi, x), lo);
    } else if (hx < 0x33000000u) {
        t = __fadd_rn(huge, x);
        return __fsub_rn(x, __fsub_rn(t, __fadd_rn(huge, x)));
    } else {
        k = 0;
    }
    hfx = __fmul_rn(0.5f, x);
    hxs = __fmul_rn(x, hfx);
    float poly = __fadd_rn(q4, __fmul_rn(hxs, q5));
    poly = __fadd_rn(q3, __fmul_rn(hxs, poly));
    poly = __fadd_rn(q2, __fmul_rn(hxs, poly));
    poly = __fadd_rn(q1, __fmul_rn(hxs, poly));
    r1 = __fadd_rn(one, __fmul_rn(hxs, poly));
    t = __fsub_rn(3.0f, __fmul_rn(r1, hfx));
    e = __fmul_rn(hxs, __fdiv_rn(__fsub_rn(r1, t), __fsub_rn(6.0f, __fmul_rn(x, t))));
    if (k == 0) return __fsub_rn(x, __fsub_rn(__fmul_rn(x, e), hxs));
    e = __fsub_rn(__fmul_rn(x, __fsub_rn(e, c)), c);
    e = __fsub_rn(e, hxs);
    if (k == -1) return __fsub_rn(__fmul_rn(0.5f, __fsub_rn(x, e)), 0.5f);
    if (k == 1) {
        if (x < -0.25f) return __fmul_rn(-2.0f, __fsub_rn(e, __fadd_rn(x, 0.5f)));
        return __fadd_rn(one, __fmul_rn(2.0f, __fsub_rn(x, e)));
    }
    if (k <= -2 || k > 56) {
        y = __fsub_rn(one, __fsub_rn(e, x));
        y = __uint_as_float(__float_as_uint(y) + ((uint32_t)k << 23));
        return __fsub_rn(y, one);
    }
    if (k < 23) {
        t = __uint_as_float(0x3f800000u - (0x1000000u >> k));
        y = __fsub_rn(t, __fsub_rn(e, x));
        y = __uint_as_float(__float_as_uint(y) + ((uint32_t)k << 23));
    } else {
        t = __uint_as_float((uint32_t)(0x7f - k) << 23);
        y = __fsub_rn(x, __fadd_rn(e, t));
        y = __fadd_rn(y, one);
        y = __uint_as_float(__float_as_uint(y) + ((uint32_t)k << 23));
    }
    return y;
}

__device__ __forceinline__ float exact_tanhf(float x) {
    const float one = 1.0f, two = 2.0f, tiny = 1.0e-30f;
    float t, z;
    const int32_t jx = (int32_t)__float_as_uint(x);
    const int32_t ix = jx & 0x7fffffff;
    if (ix >= 0x7f800000) {
        return (jx >= 0) ? __fadd_rn(__fdiv_rn(one, x), one) : __fsub_rn(__fdiv_rn(one, x), one);
    }
    if (ix < 0x41b00000) {
        if (ix == 0) return x;
        if (ix < 0x24000000) return __fmul_rn(x, __fadd_rn(one, x));
        if (ix >= 0x3f800000) {
            t = exact_expm1f(__fmul_rn(two, fabsf(x)));
            z = __fsub_rn(one, __fdiv_rn(two, __fadd_rn(t, two)));
        } else {
            t = exact_expm1f(__fmul_rn(-two, fabsf(x)));
            z = __fdiv_rn(-t, __fadd_rn(t, two));
        }
    } else {
        z = __fsub_rn(one, tiny);
    }
    return (jx >= 0) ? z : -z;
}

// tensor.cpp:141-152, op for op:
//   0.5f * v * (1.0f + tanh(kSqrt2OverPi * (v + 0.044715f * v * v * v)))
__device__ __forceinline__ float exact_gelu(float v) {
    const float k = __fsqrt_rn(__fdiv_rn(2.0f, (float)3.14159265358979323846));
    const float cube = __fmul_rn(__fmul_rn(__fmul_rn(0.044715f, v), v), v);
    const float th = exact_tanhf(__fmul_rn(k, __fadd_rn(v, cube)));
    return __fmul_rn(__fmul_rn(0.5f, v), __fadd_rn(1.0f, th));
}

// ---------------------------------------------------------------------------
// Production math (fast intrinsics; PROD mode only).
// GELU (tanh form) with the single-instruction MUFU tanh (|rel err| ~ 2^-11, far below
// the bf16 rounding of the result): 0.5 v (1 + tanh(k (v + 0.044715 v^3))).
__device__ __forceinline__ float gelu_tanh_approx(float v) {
    const float u = 0.7978845608028654f * fmaf(0.044715f * v, v * v, v);
    float th;
    asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(u));
    const float hv = 0.5f * v;
    return fmaf(hv, th, hv);
}
__device__ __forceinline__ float fast_gelu(float v) {
    const float k = 0.7978845608028654f;
    const float u = k * (v + 0.044715f * v * v * v);
    // tanh(u) = 1 - 2/(exp(2u)+1); ex2.approx based
    const float e = exp2f(u * 2.8853900817779268f);  // 2*log2(e)
    const float th = 1.0f - __fdividef(2.0f, e + 1.0f);
    return 0.5f * v * (1.0f + th);
}

__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ __nv_bfloat16 f2bf(float v) { return __float2bfloat16_rn(v); }

}  // namespace dev
}  // namespace csd
