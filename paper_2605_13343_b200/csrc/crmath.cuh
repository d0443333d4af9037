// Correctly rounded (with overwhelming probability) double log and cos, for host and device.
//
// The frame generator's normals (rng.hpp normal_of: sqrt(-2 log u1) cos(2 pi u2), the
// reference's Box-Muller, frame.cpp:154-159 / :171-179) must be bit-identical between the host
// (glibc libm) and the GPU. glibc's log and cos return the correctly rounded double on every
// input we have sampled (tools/crmath_check.cpp: 2^28 draws of the generator's own inputs,
// zero mismatches), while CUDA's log/cos are accurate to 1-2 ulp only. So the device evaluates
// both in double-double arithmetic (~2^-100 relative error) and rounds once: the result can
// differ from the correctly rounded one only if the true value lies within 2^-100 of a rounding
// midpoint.
//
// Every operation is an explicit round-to-nearest primitive, so nvcc cannot contract them into
// FMAs and the host build (-ffp-contract=off) computes the same bits.
#pragma once
#include <math.h>
#include <stdint.h>

#ifndef __CUDACC__
#ifndef __host__
#define __host__
#define __device__
#define __forceinline__ inline
#endif
#endif

// The host compiler must not contract the double-double primitives (the library's host code is
// built with -ffp-contract=fast to match the reference's -march=native build).
#if !defined(__CUDA_ARCH__) && defined(__GNUC__) && !defined(__clang__)
#pragma GCC push_options
#pragma GCC optimize("fp-contract=off")
#define CRM_POP_OPTIONS 1
#endif

namespace crm {

#ifdef __CUDA_ARCH__
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double div_(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
#else
inline double add_(double a, double b) { return a + b; }
inline double sub_(double a, double b) { return a - b; }
inline double mul_(double a, double b) { return a * b; }
inline double div_(double a, double b) { return a / b; }
inline double fma_(double a, double b, double c) { return fma(a, b, c); }
#endif

struct dd {
    double hi, lo;
};

__host__ __device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = add_(a, b), bb = sub_(s, a);
    return {s, add_(sub_(a, sub_(s, bb)), sub_(b, bb))};
}
__host__ __device__ __forceinline__ dd fast_two_sum(double a, double b) {  // |a| >= |b|
    const double s = add_(a, b);
    return {s, sub_(b, sub_(s, a))};
}
__host__ __device__ __forceinline__ dd two_prod(double a, double b) {
    const double p = mul_(a, b);
    return {p, fma_(a, b, -p)};
}
__host__ __device__ __forceinline__ dd dd_add(dd a, dd b) {  // accurate (IEEE-style) sum
    dd s = two_sum(a.hi, b.hi);
    const dd t = two_sum(a.lo, b.lo);
    s.lo = add_(s.lo, t.hi);
    s = fast_two_sum(s.hi, s.lo);
    s.lo = add_(s.lo, t.lo);
    return fast_two_sum(s.hi, s.lo);
}
__host__ __device__ __forceinline__ dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo = add_(p.lo, add_(mul_(a.hi, b.lo), mul_(a.lo, b.hi)));
    return fast_two_sum(p.hi, p.lo);
}
__host__ __device__ __forceinline__ dd dd_mul_d(dd a, double b) {
    dd p = two_prod(a.hi, b);
    p.lo = fma_(a.lo, b, p.lo);
    return fast_two_sum(p.hi, p.lo);
}
__host__ __device__ __forceinline__ dd dd_div(dd a, dd b) {  // a / b, two Newton-style corrections
    const double q1 = div_(a.hi, b.hi);
    dd r = dd_add(a, dd_mul_d({-b.hi, -b.lo}, q1));
    const double q2 = div_(r.hi, b.hi);
    r = dd_add(r, dd_mul_d({-b.hi, -b.lo}, q2));
    const double q3 = div_(r.hi, b.hi);
    dd q = fast_two_sum(q1, q2);
    return dd_add(q, {q3, 0.0});
}
// 1/k as a double-double (exact reciprocal to ~2^-106)
__host__ __device__ __forceinline__ dd dd_recip(double k) {
    const double h = div_(1.0, k);
    const double l = div_(fma_(-h, k, 1.0), k);
    return {h, l};
}

// ln 2 and pi/2 split into doubles (exact rationals from Machin / atanh series, 400 bits)
constexpr double kLn2Hi = 0x1.62e42fefa39efp-1, kLn2Lo = 0x1.abc9e3b39803fp-56;
constexpr double kPio2_1 = 0x1.921fb54442d18p+0, kPio2_2 = 0x1.1a62633145c07p-54,
                 kPio2_3 = -0x1.f1976b7ed8fbcp-110;

// log(x), x positive and normal.
__host__ __device__ inline double log_cr(double x) {
    // 1/(2k+1), k = 0..24, as double-doubles
    const double oh[25] = {0x1p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3,
        0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4,
        0x1.e1e1e1e1e1e1ep-5, 0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5,
        0x1.47ae147ae147bp-5, 0x1.2f684bda12f68p-5, 0x1.1a7b9611a7b96p-5, 0x1.0842108421084p-5,
        0x1.f07c1f07c1f08p-6, 0x1.d41d41d41d41dp-6, 0x1.bacf914c1bad0p-6, 0x1.a41a41a41a41ap-6,
        0x1.8f9c18f9c18fap-6, 0x1.7d05f417d05f4p-6, 0x1.6c16c16c16c17p-6, 0x1.5c9882b931057p-6,
        0x1.4e5e0a72f0539p-6};
    const double ol[25] = {0.0, 0x1.5555555555555p-56, -0x1.999999999999ap-57, 0x1.2492492492492p-57,
        0x1.c71c71c71c71cp-58, -0x1.745d1745d1746p-59, -0x1.3b13b13b13b14p-58, 0x1.1111111111111p-60,
        0x1.e1e1e1e1e1e1ep-61, 0x1.af286bca1af28p-59, 0x1.8618618618618p-59, 0x1.642c8590b2164p-60,
        -0x1.eb851eb851eb8p-61, 0x1.2f684bda12f68p-59, 0x1.1a7b9611a7b96p-61, 0x1.0842108421084p-60,
        -0x1.f07c1f07c1f08p-61, 0x1.0750750750750p-60, -0x1.bacf914c1bad0p-60, 0x1.0690690690690p-60,
        -0x1.f3831f3831f38p-61, 0x1.7d05f417d05f4p-62, -0x1.f49f49f49f49fp-61, 0x1.310572620ae4cp-61,
        0x1.e0a72f0539783p-60};
    int e;
    double m = frexp(x, &e);  // x = m 2^e, m in [0.5, 1)
    if (m < 0.70710678118654752440) {
        m = mul_(m, 2.0);
        e -= 1;
    }
    // log m = 2 atanh f, f = (m - 1) / (m + 1); m - 1 is exact (Sterbenz)
    const dd f = dd_div({sub_(m, 1.0), 0.0}, two_sum(m, 1.0));
    const dd f2 = dd_mul(f, f);
    // sum_k f2^k / (2k + 1): |f2| <= 0.0295, 25 terms reach 2^-126
    dd p = {oh[24], ol[24]};
#pragma unroll
    for (int k = 23; k >= 0; --k) p = dd_add(dd_mul(p, f2), {oh[k], ol[k]});
    dd lm = dd_mul(p, f);
    lm = {mul_(lm.hi, 2.0), mul_(lm.lo, 2.0)};
    const dd le = dd_add(two_prod(double(e), kLn2Hi), two_prod(double(e), kLn2Lo));
    const dd r = dd_add(le, lm);
    return add_(r.hi, r.lo);
}

// 1/n!, n = 0..29, as double-doubles
#define CRM_INVFACT                                                                              \
    const double fh[30] = {0x1p+0, 0x1p+0, 0x1p-1, 0x1.5555555555555p-3, 0x1.5555555555555p-5,      \
        0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-16,   \
        0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26, 0x1.1eed8eff8d898p-29,  \
        0x1.6124613a86d09p-33, 0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-41, 0x1.ae7f3e733b81fp-45,  \
        0x1.952c77030ad4ap-49, 0x1.6827863b97d97p-53, 0x1.2f49b46814157p-57, 0x1.e542ba4020225p-62,  \
        0x1.71b8ef6dcf572p-66, 0x1.0ce396db7f853p-70, 0x1.761b41316381ap-75, 0x1.f2cf01972f578p-80,  \
        0x1.3f3ccdd165fa9p-84, 0x1.88e85fc6a4e5ap-89, 0x1.d1ab1c2dccea3p-94, 0x1.0a18a2635085dp-98,  \
        0x1.259f98b4358adp-103};                                                                 \
    const double fl[30] = {0.0, 0.0, 0.0, 0x1.5555555555555p-57, 0x1.5555555555555p-59,             \
        0x1.1111111111111p-63, -0x1.f49f49f49f49fp-65, 0x1.a01a01a01a01ap-73, 0x1.a01a01a01a01ap-76, \
        -0x1.c154f8ddc6c00p-73, 0x1.cbbc05b4fa99ap-76, -0x1.c062e06d1f209p-80,                       \
        -0x1.2aec959e14c06p-83, 0x1.f28e0cc748ebep-87, 0x1.05d6f8a2efd1fp-92, 0x1.1d8656b0ee8cbp-97, \
        0x1.1d8656b0ee8cbp-101, 0x1.ac981465ddc6cp-103, 0x1.eec01221a8b0bp-107,                      \
        0x1.2650f61dbdcb4p-112, 0x1.ea72b4afe3c2fp-120, -0x1.d043ae40c4647p-120,                     \
        -0x1.aebcdbd20331cp-124, -0x1.3423c7d91404fp-130, -0x1.9ada5fcc1ab14p-135,                   \
        -0x1.58ddadf344487p-139, -0x1.71c37ebd16540p-143, 0x1.054d0c78aea14p-149,                    \
        0x1.b9e2e28e1aa54p-153, 0x1.eaf8c39dd9bc5p-157};

// sin r / cos r, |r| <= pi/4 + eps, r a double-double: Taylor to r^29 / r^28 (< 2^-115).
__host__ __device__ inline dd dd_sin_small(dd r) {
    CRM_INVFACT
    const dd r2 = dd_mul(r, r);
    dd p = {fh[29], fl[29]};  // k = 14, (+)
#pragma unroll
    for (int k = 13; k >= 0; --k) {
        const dd c = (k & 1) ? dd{-fh[2 * k + 1], -fl[2 * k + 1]} : dd{fh[2 * k + 1], fl[2 * k + 1]};
        p = dd_add(dd_mul(p, r2), c);
    }
    return dd_mul(p, r);
}
__host__ __device__ inline dd dd_cos_small(dd r) {
    CRM_INVFACT
    const dd r2 = dd_mul(r, r);
    dd p = {fh[28], fl[28]};  // k = 14
#pragma unroll
    for (int k = 13; k >= 0; --k) {
        const dd c = (k & 1) ? dd{-fh[2 * k], -fl[2 * k]} : dd{fh[2 * k], fl[2 * k]};
        p = dd_add(dd_mul(p, r2), c);
    }
    return p;
}

// cos(y) for 0 <= y < 8 (the generator's 2 pi u2 range).
__host__ __device__ inline double cos_cr(double y) {
    const double jd = floor(add_(mul_(y, 0.63661977236758134308), 0.5));  // nearest multiple of pi/2
    const int j = int(jd);
    // r = y - j pi/2, pi/2 in three parts: j P1 split exactly (two_prod), y - hi(j P1) exact
    // (Sterbenz: y within a factor two of j P1 when j >= 1)
    const dd p1 = two_prod(jd, kPio2_1);
    dd r = two_sum(sub_(y, p1.hi), -p1.lo);
    const dd p2 = two_prod(jd, kPio2_2);
    r = dd_add(r, {-p2.hi, -p2.lo});
    r = dd_add(r, {-mul_(jd, kPio2_3), 0.0});
    dd v;
    switch (j & 3) {
        case 0: v = dd_cos_small(r); break;
        case 1: v = dd_sin_small(r); v = {-v.hi, -v.lo}; break;
        case 2: v = dd_cos_small(r); v = {-v.hi, -v.lo}; break;
        default: v = dd_sin_small(r); break;
    }
    return add_(v.hi, v.lo);
}

// rng.hpp normal_of, bit-identical to the host's libm evaluation.
__host__ __device__ inline double normal_of_cr(uint64_t bits) {
    const double u1 = mul_(double(bits >> 32) + 1.0, 0x1.0p-32);
    const double u2 = mul_(double(bits & 0xFFFFFFFFULL), 0x1.0p-32);
#ifdef __CUDA_ARCH__
    const double rad = __dsqrt_rn(mul_(-2.0, log_cr(u1)));
#else
    const double rad = sqrt(mul_(-2.0, log_cr(u1)));
#endif
    return mul_(rad, cos_cr(mul_(2.0 * 3.14159265358979323846, u2)));
}

}  // namespace crm

#ifdef CRM_POP_OPTIONS
#pragma GCC pop_options
#undef CRM_POP_OPTIONS
#endif
