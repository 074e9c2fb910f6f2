// cfust_special.cuh — compact, branch-free FP64 standard-normal CDF and quantile for the SOV
// hot loop.
//
// libdevice's normcdfinv is ~600 SASS instructions with several branches; inlined at every SOV
// step it thrashed the instruction cache (ncu: stall "no_instruction" 8.1 per issue,
// profiles/r01_*).  These are single rational approximations fitted by scripts/fit_special.py
// (relative error <= 1.3e-15 in double evaluation; coefficients in cfust_coeffs.h, all positive
// so Horner has no cancellation), one formula over the whole range so a warp never diverges:
//   Phi(x):       t = exp(-x^2/2) R(|x|),  Phi = t (x < 0) or 1 - t (x >= 0)
//   Phi^{-1}(u):  t = min(u, 1-u), w = -log(2t), z = -w U(sqrt(w)), sign by u < 1/2
// Polynomials by Horner (Estrin optional); divisions by rcp.approx + Newton (no IEEE slow-path branch).
#pragma once
#include <cuda_runtime.h>

#ifndef CFUST_HORNER
#define CFUST_HORNER 1   // measured faster than Estrin on B200 (profiles/r01_variants.log)
#endif

namespace cfust {
#include "cfust_coeffs.h"

template <int N>
__device__ __forceinline__ double horner_c(const double (&c)[N], double x) {
    double r = c[N - 1];
#pragma unroll
    for (int k = N - 2; k >= 0; --k) r = fma(r, x, c[k]);
    return r;
}

// Estrin's scheme (N <= 16 coefficients): dependency depth 4 instead of N-1 for Horner; the
// powers x^2, x^4, x^8 are shared by numerator and denominator.
template <int N>
__device__ __forceinline__ double estrin_c(const double (&c)[N], double x, double x2, double x4, double x8) {
    static_assert(N <= 16, "estrin_c: up to degree 15");
    constexpr int N1 = (N + 1) / 2, N2 = (N1 + 1) / 2, N3 = (N2 + 1) / 2;
    double p1[N1], p2[N2], p3[N3];
#pragma unroll
    for (int i = 0; i < N1; ++i) p1[i] = (2 * i + 1 < N) ? fma(c[2 * i + 1], x, c[2 * i]) : c[2 * i];
#pragma unroll
    for (int i = 0; i < N2; ++i) p2[i] = (2 * i + 1 < N1) ? fma(p1[2 * i + 1], x2, p1[2 * i]) : p1[2 * i];
#pragma unroll
    for (int i = 0; i < N3; ++i) p3[i] = (2 * i + 1 < N2) ? fma(p2[2 * i + 1], x4, p2[2 * i]) : p2[2 * i];
    if constexpr (N3 == 1) return p3[0];
    else return fma(p3[1], x8, p3[0]);
}

// p / q for q > 0 normal: MUFU reciprocal seed + two Newton steps + one residual correction.
__device__ __forceinline__ double div_fast(double p, double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    double e = fma(-q, r, 1.0);
    r = fma(r, e, r);
    e = fma(-q, r, 1.0);
    r = fma(r, e, r);
    const double y = p * r;
    return fma(fma(-q, y, p), r, y);
}

#ifndef CFUST_OWN_ELEM
#define CFUST_OWN_ELEM 0   // 1: own branch-free exp/log/sqrt (measured equal speed, more registers)
#endif

// exp(x) for x <= 0 (x >= -708 exact to ~1 ulp; below: 0, i.e. results < 1e-307 flush).
// x = k ln2 + r, |r| <= ln2/2: k from the 1.5*2^52 rounding trick, r with a two-part ln2,
// Taylor to r^13, 2^k by adding k to the exponent field.
__device__ __forceinline__ double exp_neg(double x) {
#if CFUST_OWN_ELEM
    const double t = fma(x, 1.4426950408889634074, 6755399441055744.0);
    const int k = __double2loint(t);
    const double kd = t - 6755399441055744.0;
    const double r = fma(kd, -2.3190468138462996e-17, fma(kd, -0.69314718055994528623, x));
    const double p = horner_c(c_EXPC, r);
    const double res = __hiloint2double(__double2hiint(p) + k * (1 << 20), __double2loint(p));
    return (x < -708.0) ? 0.0 : res;
#else
    return exp(x);
#endif
}

// log(x) for normal x in (0, 1]: x = m 2^e, m in [sqrt(1/2), sqrt(2)); log m = 2 atanh(s),
// s = (m-1)/(m+1) (m-1 exact), series to s^21.  Relative accuracy holds as x -> 1 (e = 0).
__device__ __forceinline__ double log_unit(double x) {
#if CFUST_OWN_ELEM
    const int hx = __double2hiint(x);
    int e = (hx >> 20) - 1023;
    int mh = (hx & 0x000fffff) | 0x3ff00000;
    const bool big = mh > 0x3ff6a09e;   // m > sqrt(2): halve
    mh = big ? mh - 0x00100000 : mh;
    e = big ? e + 1 : e;
    const double m = __hiloint2double(mh, __double2loint(x));
    const double s = div_fast(m - 1.0, m + 1.0);
    const double ls = s * horner_c(c_LOGC, s * s);
    const double ed = double(e);
    return fma(ed, 0.69314718055994528623, fma(ed, 2.3190468138462996e-17, ls));
#else
    return log(x);
#endif
}

// sqrt(w), w >= 0 finite: rsqrt seed + two Newton steps + one residual correction.
__device__ __forceinline__ double sqrt_fast(double w) {
#if CFUST_OWN_ELEM
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(w));
    y = y * fma(-0.5 * w * y, y, 1.5);
    y = y * fma(-0.5 * w * y, y, 1.5);
    double v = w * y;
    v = fma(0.5 * y, fma(-v, v, w), v);
    return (w > 0.0) ? v : 0.0;
#else
    return sqrt(w);
#endif
}

// Phi(x) = P(X <= x), X ~ N(0,1); relative accuracy in the lower tail (to ~1e-307), absolute
// accuracy for x > 0.  x^2 is split exactly (hi + lo) so the exponent carries no rounding.
__device__ __forceinline__ double Phi_fast(double x) {
    const double fx = fabs(x);
    const double ax = (fx < 40.0) ? fx : 40.0;   // exp(-800) = 0: Phi is exactly 0 or 1 beyond
    const double hi = ax * ax;
    const double lo = fma(ax, ax, -hi);
    const double e = exp_neg(-0.5 * hi) * (1.0 - 0.5 * lo);
#if CFUST_HORNER
    const double t = e * div_fast(horner_c(c_PH_P, ax), horner_c(c_PH_Q, ax));
#else
    const double x4 = hi * hi, x8 = x4 * x4;
    const double t = e * div_fast(estrin_c(c_PH_P, ax, hi, x4, x8), estrin_c(c_PH_Q, ax, hi, x4, x8));
#endif
    return (x < 0.0) ? t : 1.0 - t;
}

// Phi^{-1}(u), 0 < u < 1.  1 - u is exact for u >= 1/2; 2t is exact; log(2t) is accurate to
// ~1 ulp of its value, so w keeps full relative precision as u -> 1/2.
__device__ __forceinline__ double Phiinv_fast(double u) {
    const double uc = 1.0 - u;
    const double t = (u < uc) ? u : uc;
    const double w = -log_unit(2.0 * t);
    const double v = sqrt_fast(w);
#if CFUST_HORNER
    const double z = w * div_fast(horner_c(c_NI_P, v), horner_c(c_NI_Q, v));
#else
    const double v2 = v * v, v4 = v2 * v2, v8 = v4 * v4;
    const double z = w * div_fast(estrin_c(c_NI_P, v, v2, v4, v8), estrin_c(c_NI_Q, v, v2, v4, v8));
#endif
    return (u < 0.5) ? -z : z;
}

}  // namespace cfust
