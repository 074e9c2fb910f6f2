// cfust_special.cuh — compact, branch-free FP64 standard-normal CDF and quantile for the SOV
// hot loop.
//
// libdevice's normcdfinv is ~600 SASS instructions with several branches; inlined at every SOV
// step it thrashed the instruction cache (ncu: stall "no_instruction" 8.1 per issue,
// profiles/r01_*).  These are single rational approximations fitted by scripts/fit_special.py
// (relative error <= 1.3e-15 in double evaluation; Mills ratio (9,10); coefficients in cfust_coeffs.h, all positive
// so Horner has no cancellation), one formula over the whole range so a warp never diverges:
//   Phi(x):       t = exp(-x^2/2) R(|x|),  Phi = t (x < 0) or 1 - t (x >= 0)
//   Phi^{-1}(u):  t = min(u, 1-u), FP32 seed z0 ~ -w U(sqrt(w)) (w = -log(2t)), then one
//                 third-order FP64 correction through Phi's own rational (Phiinv_seed, default);
//                 Phiinv_rat (the FP64 (14,15) rational in sqrt(w)) is kept for comparison.
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

#ifndef CFUST_DIV_NEWTON
#define CFUST_DIV_NEWTON 1   // Newton steps on the reciprocal before the quotient correction
#endif
// p / q for normal q: MUFU reciprocal seed (relative error e0 ~ 2^-22), CFUST_DIV_NEWTON Newton
// steps on 1/q (one: e0^2 ~ 1e-13), then the residual correction y + r (p - q y), itself a Newton
// step on the quotient: error ~ e1^2 + rounding, i.e. within an ulp (tests/test_gpu_special.py).
__device__ __forceinline__ double div_fast(double p, double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
#pragma unroll
    for (int k = 0; k < CFUST_DIV_NEWTON; ++k) {
        const double e = fma(-q, r, 1.0);
        r = fma(r, e, r);
    }
    const double y = p * r;
    return fma(fma(-q, y, p), r, y);
}

#ifndef CFUST_DIV_F32
#define CFUST_DIV_F32 0   // 1: Phi's quotient from an FP32 reciprocal seed (two FP64 Newton steps)
#endif
// P / Q for the Mills-ratio rational only (Q in [1, 1e11] on [0, 40]: safe in FP32).
__device__ __forceinline__ double div_rat(double p, double q) {
#if CFUST_DIV_F32
    float rf;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rf) : "f"(__double2float_rn(q)));
    double r = double(rf);
    double e = fma(-q, r, 1.0);
    r = fma(r, e, r);
    e = fma(-q, r, 1.0);
    r = fma(r, e, r);
    const double y = p * r;
    return fma(fma(-q, y, p), r, y);
#else
    return div_fast(p, q);
#endif
}

#ifndef CFUST_HORNER_EO
#define CFUST_HORNER_EO 0   // 1: even/odd split Horner (two half-length chains per polynomial)
#endif
// p(x) = pe(x^2) + x po(x^2) with x2 = x*x supplied by the caller.
template <int N>
__device__ __forceinline__ double horner_eo(const double (&c)[N], double x, double x2) {
#if CFUST_HORNER_EO
    constexpr int NE = (N + 1) / 2, NO = N / 2;
    double pe = c[2 * (NE - 1)];
#pragma unroll
    for (int k = NE - 2; k >= 0; --k) pe = fma(pe, x2, c[2 * k]);
    double po = c[2 * (NO - 1) + 1];
#pragma unroll
    for (int k = NO - 2; k >= 0; --k) po = fma(po, x2, c[2 * k + 1]);
    return fma(po, x, pe);
#else
    (void)x2;
    return horner_c(c, x);
#endif
}

#ifndef CFUST_OWN_ELEM
#define CFUST_OWN_ELEM 1   // own branch-free exp/log/sqrt; with the seeded Phi^{-1} 11% faster E-step
#endif                     // than libdevice (profiles/r01_seed_variants.log)

#ifndef CFUST_INTSEL
#define CFUST_INTSEL 0   // 1: sign / range tests on the integer image of the double (INT pipe, not DSETP)
#endif

#ifndef CFUST_EXP_TAB
#define CFUST_EXP_TAB 0
#endif

// 2^(j/64), j = 0..63, correctly rounded (mpmath, 200 bits): exp by table (CFUST_EXP_TAB through
// L1, and the q = 0 kernel from a shared-memory copy).
__device__ const double g_EXP2J[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0,
};

// exp(x) for x <= 709 (x >= -708 exact to ~1 ulp; below: 0, i.e. results < 1e-307 flush).
// Default: x = k ln2 + r, |r| <= ln2/2: k from the 1.5*2^52 rounding trick, r with a two-part
// ln2, near-minimax degree-11 polynomial (c_EXPC, scripts/fit_special.py), 2^k by adding k to the
// exponent field.
// CFUST_EXP_TAB: x = (64 m + j) ln2/64 + r, |r| <= ln2/128: exp = 2^m 2^(j/64) (1 + q(r)),
// q = r + ... + r^5/120 (truncation r^6/720 < 4e-17), 2^(j/64) from a 64-entry table:
// 10 FP64 operations instead of 17.
__device__ __forceinline__ double exp_neg(double x) {
#if CFUST_OWN_ELEM && CFUST_EXP_TAB
    const double t = fma(x, 92.33248261689366, 6755399441055744.0);
    const int k = __double2loint(t);
    const double kd = t - 6755399441055744.0;
    const double r = fma(kd, -3.623510646634843e-19, fma(kd, -0.010830424696249145, x));
    const double q = r * fma(r, fma(r, fma(r, fma(r, 1.0 / 120.0, 1.0 / 24.0), 1.0 / 6.0), 0.5), 1.0);
    const double T = __ldg(&g_EXP2J[k & 63]);
    const double p = fma(T, q, T);
    const double res = __hiloint2double(__double2hiint(p) + (k >> 6) * (1 << 20), __double2loint(p));
    return (x < -708.0) ? 0.0 : res;
#elif CFUST_OWN_ELEM
    const double t = fma(x, 1.4426950408889634074, 6755399441055744.0);
    const int k = __double2loint(t);
    const double kd = t - 6755399441055744.0;
    const double r = fma(kd, -2.3190468138462996e-17, fma(kd, -0.69314718055994528623, x));
    const double p = horner_c(c_EXPC, r);
    const double res = __hiloint2double(__double2hiint(p) + k * (1 << 20), __double2loint(p));
#if CFUST_INTSEL
    // x < -708 <=> negative with |x| > 708: unsigned high word above that of -708 (0xC0862000); the
    // few doubles in (-708 - 2^-43, -708) pass through and get their (normal, accurate) value
    return (unsigned(__double2hiint(x)) > 0xC0862000u) ? 0.0 : res;
#else
    return (x < -708.0) ? 0.0 : res;
#endif
#else
    return exp(x);
#endif
}

// exp(xh + xl) for |xl| << 1 ulp-scale of xh (the low part of an exact square): xl joins the reduced
// argument r, where it is representable, instead of a separate (1 + xl) factor (one op fewer).
__device__ __forceinline__ double exp_neg2(double xh, double xl) {
#if CFUST_OWN_ELEM && !CFUST_EXP_TAB
    const double t = fma(xh, 1.4426950408889634074, 6755399441055744.0);
    const int k = __double2loint(t);
    const double kd = t - 6755399441055744.0;
    const double r = fma(kd, -2.3190468138462996e-17, fma(kd, -0.69314718055994528623, xh)) + xl;
    const double p = horner_eo(c_EXPC, r, r * r);
    const double res = __hiloint2double(__double2hiint(p) + k * (1 << 20), __double2loint(p));
    return (xh < -708.0) ? 0.0 : res;
#else
    return exp_neg(xh) * (1.0 + xl);
#endif
}

// log(x) for normal x > 0: x = m 2^e, m in [sqrt(1/2), sqrt(2)); log m = 2 atanh(s),
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

// log(1 + x), x >= 0: log of z = 1 + x (log_unit handles any positive normal z) plus the
// rounding correction (x - (z - 1)) / z (a tiny term: an approximate reciprocal suffices).
__device__ __forceinline__ double log1p_pos(double x) {
    const double z = 1.0 + x;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(z));
    return fma(x - (z - 1.0), r, log_unit(z));
}

// Table-driven log and exp for the q = 0 E-step (tables in shared memory, filled per block):
//   log z = e ln2 - log(invc_j) + log1p(r),  r = m invc_j - 1 (one rounding, |r| < 2^-7),
//     j = the top 7 mantissa bits, invc_j = RN(1 / (1 + (j + 1/2)/128)) (j = 0: exactly 1, so that
//     log z -> 0 keeps its relative accuracy), log1p(r) to r^8 (relative truncation < 2e-18);
//   exp x = 2^m 2^(j/64) e^r,  x = (64 m + j) ln2/64 + r, |r| <= ln2/128, e^r - 1 to r^6 (< 3e-20).
// About 12 FP64 operations each instead of ~20 (log: division + degree-21 series) / 17 (exp).
__device__ __forceinline__ double log_tab(double z, const double2 *__restrict__ tab) {
    const int hz = __double2hiint(z);
    const int e = (hz >> 20) - 1023;
    const double m = __hiloint2double((hz & 0x000fffff) | 0x3ff00000, __double2loint(z));
    const double2 t = tab[(hz >> 13) & 127];
    const double r = fma(m, t.x, -1.0);
    const double poly = fma(r, fma(r, fma(r, fma(r, fma(r, fma(r, -0.125, 1.0 / 7), -1.0 / 6), 1.0 / 5), -0.25), 1.0 / 3), -0.5);
    const double ed = double(e);
    return fma(ed, 0.69314718055994528623, t.y) + fma(ed, 2.3190468138462996e-17, fma(r * r, poly, r));
}
// log(1 + x), x >= 0, with the rounding correction of 1 + x (as log1p_pos)
__device__ __forceinline__ double log1p_tab(double x, const double2 *__restrict__ tab) {
    const double z = 1.0 + x;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(z));
    return fma(x - (z - 1.0), r, log_tab(z, tab));
}
// exp(x) for x <= 0 (x < -708: 0)
__device__ __forceinline__ double exp_tab(double x, const double *__restrict__ tab) {
    const double t = fma(x, 92.33248261689366, 6755399441055744.0);   // 64 / ln2, round to integer k
    const int k = __double2loint(t);
    const double kd = t - 6755399441055744.0;
    const double r = fma(kd, -3.623510646634843e-19, fma(kd, -0.010830424696249145, x));   // x - k ln2/64
    const double q = r * fma(r, fma(r, fma(r, fma(r, fma(r, 1.0 / 720, 1.0 / 120), 1.0 / 24), 1.0 / 6), 0.5), 1.0);
    const double T = tab[k & 63];
    const double p = fma(T, q, T);
    const double res = __hiloint2double(__double2hiint(p) + (k >> 6) * (1 << 20), __double2loint(p));
    return (x < -708.0) ? 0.0 : res;
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

// exp(xh + xl) (as exp_neg2) with 2^(j/64) from the 64-entry table through L1:
// x = (64 m + j) ln2/64 + r, |r| <= ln2/128, e^r - 1 to r^5/120 (truncation < 4e-17): 9 FP64
// operations and one table load (off the dependent chain: the load runs beside the polynomial)
// instead of the 16 of the degree-11 polynomial.  The SOV loop of the kernel CFUST_SOV_XT = q uses
// it (Tune<q>::XT; off by default: -1.3 % at q = 3, +1.3 % at q = 2, profiles/r02w_ab.log).
__device__ __forceinline__ double exp_tab2(double xh, double xl) {
    const double t = fma(xh, 92.33248261689366, 6755399441055744.0);   // 64 / ln2, round to integer k
    const int k = __double2loint(t);
    const double kd = t - 6755399441055744.0;
    const double r = fma(kd, -3.623510646634843e-19, fma(kd, -0.010830424696249145, xh)) + xl;
    const double T = __ldg(&g_EXP2J[k & 63]);
    const double q = r * fma(r, fma(r, fma(r, fma(r, 1.0 / 120.0, 1.0 / 24.0), 1.0 / 6.0), 0.5), 1.0);
    const double p = fma(T, q, T);
    const double res = __hiloint2double(__double2hiint(p) + (k >> 6) * (1 << 20), __double2loint(p));
    return (xh < -708.0) ? 0.0 : res;
}
template <bool XT>
__device__ __forceinline__ double exp_sov(double xh, double xl) {
    if constexpr (XT) return exp_tab2(xh, xl);
    else return exp_neg2(xh, xl);
}

// Phi(x) = P(X <= x), X ~ N(0,1); relative accuracy in the lower tail (to ~1e-307), absolute
// accuracy for x > 0.  x^2 is split exactly (hi + lo) so the exponent carries no rounding.
// XT: exp by table (exp_tab2).
template <bool XT>
__device__ __forceinline__ double Phi_x(double x) {
    const double fx = fabs(x);
    const double ax = (fx < 40.0) ? fx : 40.0;   // exp(-800) = 0: Phi is exactly 0 or 1 beyond
    const double hi = ax * ax;
    const double lo = fma(ax, ax, -hi);
    const double e = exp_sov<XT>(-0.5 * hi, -0.5 * lo);
#if CFUST_HORNER
    const double t = e * div_rat(horner_eo(c_PH_P, ax, hi), horner_eo(c_PH_Q, ax, hi));
#else
    const double x4 = hi * hi, x8 = x4 * x4;
    const double t = e * div_fast(estrin_c(c_PH_P, ax, hi, x4, x8), estrin_c(c_PH_Q, ax, hi, x4, x8));
#endif
#if CFUST_INTSEL
    return (__double2hiint(x) < 0) ? t : 1.0 - t;   // sign bit (x = -0: t = 1/2 either way)
#else
    return (x < 0.0) ? t : 1.0 - t;
#endif
}
__device__ __forceinline__ double Phi_fast(double x) { return Phi_x<false>(x); }

// Phi^{-1}(u), 0 < u < 1.  1 - u is exact for u >= 1/2; 2t is exact; log(2t) is accurate to
// ~1 ulp of its value, so w keeps full relative precision as u -> 1/2.
__device__ __forceinline__ double Phiinv_rat(double u) {
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

// FP32 MUFU approximations with flush-to-zero (no subnormal pre-scaling instructions; the
// arguments here are never subnormal).
__device__ __forceinline__ float lg2_ftz(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// FP32 seed of the lower-tail quantile U(v) ~ Phi^{-1}(t) = -w U(sqrt w), w = -log(2t):
// rational (8, 8) in v fitted by scripts/fit_special.py --seed (relative error 4.4e-7 in FP32
// evaluation); literals, so FFMA takes them as immediates.
__device__ __forceinline__ float seed_U32(float v) {
    float p = -1.1203700189810206e-09f;
    p = fmaf(p, v, 0.0089739840477705f);
    p = fmaf(p, v, 0.2872512638568878f);
    p = fmaf(p, v, 2.012030839920044f);
    p = fmaf(p, v, 4.561682224273682f);
    p = fmaf(p, v, 6.014867305755615f);
    p = fmaf(p, v, 5.465461254119873f);
    p = fmaf(p, v, 3.105163097381592f);
    p = fmaf(p, v, 1.2533141374588013f);
    float q = 0.006345330271869898f;
    q = fmaf(q, v, 0.20316024124622345f);
    q = fmaf(q, v, 1.4386792182922363f);
    q = fmaf(q, v, 3.551027536392212f);
    q = fmaf(q, v, 5.64398193359375f);
    q = fmaf(q, v, 6.0376763343811035f);
    q = fmaf(q, v, 4.860823631286621f);
    q = fmaf(q, v, 2.4775614738464355f);
    q = fmaf(q, v, 1.0f);
    return p * rcp_ftz(q);
}

// Phi^{-1}(u), 0 < u < 1, by an FP32 seed and one third-order FP64 correction.
//   t = min(u, 1-u) <= 1/2 (exact), z0 = -w U32(sqrt w) in FP32 from w = -log(2t) (exponent and
//   20 mantissa bits of t; |error| <= ~5e-7 |z0| + 1e-7), then with the FP64 Mills-ratio rational
//   R of Phi_fast (Phi(z0) = e^{-z0^2/2} R(|z0|)) and the exact derivatives of the inverse
//   (x' = 1/phi, x'' = x/phi^2, x''' = (1 + 2x^2)/phi^3):
//     r = (t - Phi(z0)) / phi(z0) = sqrt(2 pi) (t e^{z0^2/2} - R(|z0|)),
//     x = z0 + r + (z0/2) r^2 + ((1 + 2 z0^2)/6) r^3      (truncation ~ (z0^3/4) r^4 < 1e-16 |x|).
//   No log, no sqrt, one division in FP64 (vs log + sqrt + a (14,15) rational + division).
//   Accuracy (CPU emulation, tests/test_special_coeffs.py): relative 3e-16 for |x| >= 1,
//   absolute 4e-16 below (the SOV loop consumes z only through a = s b - sum C z).
template <bool XT>
__device__ __forceinline__ double Phiinv_seed_x(double u) {
    const double uc = 1.0 - u;
    const double t = (u < uc) ? u : uc;
    const int hx = __double2hiint(t);
    const float m = __int_as_float(0x3f800000 | ((hx & 0x000fffff) << 3));   // mantissa of t in [1,2)
    const float e2t = float((hx >> 20) - 1022);                             // 2t = m 2^e2t
    float w = -0.6931471806f * (e2t + lg2_ftz(m));
    w = fmaxf(w, 0.0f);
    const float v = (w > 0.0f) ? w * rsqrt_ftz(w) : 0.0f;
    const double ax = fmin(double(w * seed_U32(v)), 37.5);                   // |z0|
    const double hi = ax * ax;
    const double lo = fma(ax, ax, -hi);
    const double ep = exp_sov<XT>(0.5 * hi, 0.5 * lo);                      // e^{z0^2/2} (valid to +709)
    const double R = div_rat(horner_eo(c_PH_P, ax, hi), horner_eo(c_PH_Q, ax, hi));
    const double r = 2.5066282746310002 * fma(t, ep, -R);
    const double x = fma(r, fma(r, fma(r, fma(hi, 1.0 / 3.0, 1.0 / 6.0), -0.5 * ax), 1.0), -ax);
#if CFUST_INTSEL
    return (__double2hiint(u) < 0x3FE00000) ? x : -x;   // u in (0, 1): u < 1/2 <=> high word below 0.5's
#else
    return (u < 0.5) ? x : -x;
#endif
}
__device__ __forceinline__ double Phiinv_seed(double u) { return Phiinv_seed_x<false>(u); }

// u clamped to [UMIN, UMAX] for u >= 0 (u = w e with w, e in [0, 1]); with CFUST_INTSEL on the
// integer image (non-negative doubles order like their bit patterns).
__device__ __forceinline__ double clamp_u(double u, double lo, double hi) {
#if CFUST_INTSEL
    long long b = __double_as_longlong(u);
    const long long bl = __double_as_longlong(lo), bh = __double_as_longlong(hi);
    b = (b < bl) ? bl : b;
    b = (b > bh) ? bh : b;
    return __longlong_as_double(b);
#else
    u = (u < lo) ? lo : u;   // plain compares, no NaN semantics
    return (u > hi) ? hi : u;
#endif
}

#ifndef CFUST_PHIINV_SEED
#define CFUST_PHIINV_SEED 1
#endif
__device__ __forceinline__ double Phiinv_fast(double u) {
#if CFUST_PHIINV_SEED
    return Phiinv_seed(u);
#else
    return Phiinv_rat(u);
#endif
}

}  // namespace cfust
