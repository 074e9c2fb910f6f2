// cfust_device.cuh — device-side data layout and FP64 special functions (sm_100a).
//
// Independent of oracle/ (no shared code): written for the GPU from the same mathematical
// definitions.  Cites: Eq. (2) PAPER.md:154-166.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "cfust_special.cuh"

namespace cfust {

constexpr int PMAX = 8;
constexpr int QMAX = 6;
constexpr int GMAX = 8;
constexpr double UMIN = 1e-300;                 // SOV clamp (reading A15)
constexpr double UMAX = 0x1.fffffffffffffp-1;   // largest double below 1

// Per-component quantities derived from Psi, recomputed after each M-step.
struct CompDev {
    double mu[PMAX];
    double L[PMAX * PMAX];        // chol(Omega), lower, row-major p x p (stride PMAX)
    double Linv[PMAX];            // 1 / L_aa
    double A[QMAX * PMAX];        // Delta' Omega^{-1}, q x p (stride PMAX)
    double Lam[QMAX * QMAX];      // Lambda = I - Delta' Omega^{-1} Delta, q x q (stride QMAX)
    double nu, m0, kappa, logpi;  // kappa = log t_p normaliser incl. -1/2 log|Omega|
    double psi_half_m0;           // digamma(m0/2) for e1 - e2 (reading A5)
    double lgc_m0;                // lgamma((m0+1)/2) - lgamma(m0/2)      (t_1 density, df m0)
    double lgc_m0m1;              // lgamma(m0/2) - lgamma((m0-1)/2)      (t_1 density, df m0-1)
    double lbt[3];                // log B(m/2, 1/2) at m = m0, m0+1, m0+2  (t_1 CDFs of T_1 terms)
    double inv_nu;                // 1 / nu
    double log_half_nu;           // log(nu / 2)
};

struct LatticeDev {
    int M;                        // power of two
    uint32_t z[QMAX + 1];         // q + 1 coordinates for the SOV-direct estimator (reading D1)
    double shift[QMAX + 1];
};

// ------------------------------------------------------------------------------------------
// Lattice point coordinate k of point l:  x = frac((l z_k mod M)/M + shift_k), w = |2x - 1|
// (reading A11, tent periodisation).  (l z_k mod M)/M and 2x are exact in FP64.
__device__ __forceinline__ double lattice_w(const LatticeDev& L, int l, int k) {
    const uint32_t t = (uint32_t(l) * L.z[k]) & uint32_t(L.M - 1);
    double x = __dadd_rn(__dmul_rn(double(t), 1.0 / double(L.M)), L.shift[k]);
    if (x >= 1.0) x -= 1.0;
    return fabs(__dadd_rn(__dmul_rn(2.0, x), -1.0));
}

// ------------------------------------------------------------------------------------------
// Standard normal CDF / quantile used by the SOV loop (cfust_special.cuh).
__device__ __forceinline__ double Phi(double x) { return Phi_fast(x); }
__device__ __forceinline__ double Phiinv(double u) { return Phiinv_fast(u); }
// The SOV loop's copies: XT = exp by the 2^(j/64) table (exp_tab2), chosen per kernel (Tune<Q>::XT).
template <bool XT>
__device__ __forceinline__ double Phi_t(double x) { return Phi_x<XT>(x); }
template <bool XT>
__device__ __forceinline__ double Phiinv_t(double u) {
#if CFUST_PHIINV_SEED
    return Phiinv_seed_x<XT>(u);
#else
    return Phiinv_rat(u);
#endif
}

// digamma and trigamma for x > 0: upward recurrence to x >= 10, then the Stirling-type asymptotic
// series through the B_16 (digamma) / B_18 (trigamma) terms (truncation < 1e-17 relative at x = 10).
// The recurrence sums  sum_k 1/(x+k)  and  sum_k 1/(x+k)^2  are accumulated as fractions num/den,
// two steps per iteration (1/x + 1/(x+1) = (2x+1)/(x(x+1))), which halves the dependent chain of the
// M-step's nu root (one serial Newton chain per component, tests/test_gpu_special.py for accuracy).
__device__ __forceinline__ double digamma_asym(double x) {   // x >= 10
    const double r = div_fast(1.0, x), r2 = r * r;
    const double ser = r2 * (1.0 / 12 - r2 * (1.0 / 120 - r2 * (1.0 / 252 - r2 * (1.0 / 240 - r2 * (1.0 / 132
                      - r2 * (691.0 / 32760 - r2 * (1.0 / 12 - r2 * (3617.0 / 8160))))))));
    return log_unit(x) - 0.5 * r - ser;
}
__device__ __forceinline__ double trigamma_asym(double x) {   // x >= 10
    const double r = div_fast(1.0, x), r2 = r * r;
    return r * (1.0 + r * (0.5 + r * (1.0 / 6 - r2 * (1.0 / 30 - r2 * (1.0 / 42 - r2 * (1.0 / 30 - r2 * (5.0 / 66
           - r2 * (691.0 / 2730 - r2 * (7.0 / 6 - r2 * (3617.0 / 510 - r2 * (43867.0 / 798)))))))))));
}
__device__ inline double dev_digamma(double x) {
    double num = 0.0, den = 1.0;
    while (x < 9.0) {   // num/den += 1/x + 1/(x+1)
        const double t = x * (x + 1.0);
        num = fma(num, t, den * fma(2.0, x, 1.0));
        den *= t;
        x += 2.0;
    }
    if (x < 10.0) { num = fma(num, x, den); den *= x; x += 1.0; }
    return digamma_asym(x) - div_fast(num, den);
}
__device__ inline double dev_trigamma(double x) {
    double num = 0.0, den = 1.0;
    while (x < 9.0) {   // num/den += 1/x^2 + 1/(x+1)^2
        const double x2 = x * x, x12 = (x + 1.0) * (x + 1.0), t = x2 * x12;
        num = fma(num, t, den * (x2 + x12));
        den *= t;
        x += 2.0;
    }
    if (x < 10.0) { const double x2 = x * x; num = fma(num, x2, den); den *= x2; x += 1.0; }
    return div_fast(num, den) + trigamma_asym(x);
}
// both at once (the nu Newton step needs psi and psi'): the two recurrences interleave
__device__ inline void dev_psi01(double x, double &psi, double &psi1) {
    double nd = 0.0, dd = 1.0, nt = 0.0, dt = 1.0;
    while (x < 9.0) {
        const double t = x * (x + 1.0), x2 = x * x, x12 = (x + 1.0) * (x + 1.0), u = x2 * x12;
        nd = fma(nd, t, dd * fma(2.0, x, 1.0));
        dd *= t;
        nt = fma(nt, u, dt * (x2 + x12));
        dt *= u;
        x += 2.0;
    }
    if (x < 10.0) {
        nd = fma(nd, x, dd); dd *= x;
        const double x2 = x * x;
        nt = fma(nt, x2, dt); dt *= x2;
        x += 1.0;
    }
    psi = digamma_asym(x) - div_fast(nd, dd);
    psi1 = div_fast(nt, dt) + trigamma_asym(x);
}

// log Gamma(x), x > 0 (the M-step's derived constants): upward recurrence to y = x + n >= 10 as one
// product, then Stirling's series through the B_16 term (truncation < 4e-17 at y = 10):
//   lgamma(x) = (y - 1/2) log y - y + log(2 pi)/2 + sum_k B_2k / (2k (2k-1) y^(2k-1)) - log(x (x+1) ... (x+n-1)).
// One code path for every argument (libdevice lgamma branches by range: lanes with different ranges
// run one after another); absolute error ~1e-15 (tests/test_gpu_special.py).
__device__ inline double dev_lgamma_pos(double x) {
    double prod = 1.0;
    while (x < 10.0) { prod *= x; x += 1.0; }
    const double r = div_fast(1.0, x), r2 = r * r;
    const double ser = r * (1.0 / 12 - r2 * (1.0 / 360 - r2 * (1.0 / 1260 - r2 * (1.0 / 1680 - r2 * (1.0 / 1188
                       - r2 * (691.0 / 360360 - r2 * (1.0 / 156 - r2 * (3617.0 / 122400))))))));
    return fma(x - 0.5, log_unit(x), 0.91893853320467274178 - x) + ser - log_unit(prod);
}

// Continued fractions by the fundamental (Wallis) recurrences
//   A_n = b_n A_{n-1} + a_n A_{n-2},  B_n = b_n B_{n-1} + a_n B_{n-2},  K_n = A_n / B_n,
// with (A, B) rescaled by a power of two when |B_n| leaves [2^-400, 2^400].  Convergence is tested
// without a division per step: |A_n B_{n-1} - A_{n-1} B_n| <= 1e-16 |A_n B_{n-1}|.
//
// Incomplete beta (DLMF 8.17.22): I_x(a,b) = x^a (1-x)^b / (a B(a,b)) * cf,
//   cf = 1/(1 + d_1/(1 + d_2/(1 + ...))), d_{2m} = m(b-m)x/((a+2m-1)(a+2m)),
//   d_{2m+1} = -(a+m)(a+b+m)x/((a+2m)(a+2m+1)); fast for x < (a+1)/(a+b+2).
__device__ __forceinline__ void wallis_step(double an, double bn, double &A1, double &A2, double &B1, double &B2) {
    const double A = fma(bn, A1, an * A2), B = fma(bn, B1, an * B2);
    A2 = A1; B2 = B1; A1 = A; B1 = B;
    const double mb = fabs(B1);
    if (mb > 0x1p400 || mb < 0x1p-400) {
        const double s = (mb > 0x1p400) ? 0x1p-400 : 0x1p400;
        A1 *= s; B1 *= s; A2 *= s; B2 *= s;
    }
}
__device__ inline double dev_betacf(double a, double b, double x) {
    // n = 1: a_1 = 1, b_1 = 1  ->  A = 1, B = 1
    double A2 = 0.0, B2 = 1.0, A1 = 1.0, B1 = 1.0;
    for (int m = 1; m <= 4000; ++m) {
        const double k2 = 2.0 * m;
        const double de = m * (b - m) * x * div_fast(1.0, (a + k2 - 1.0) * (a + k2));          // d_{2m}
        const double d_o = -(a + m) * (a + b + m) * x * div_fast(1.0, (a + k2) * (a + k2 + 1.0));   // d_{2m+1}
        // d_{2m-1} was applied in the previous round (d_1 at m = 1 below)
        if (m == 1) wallis_step(-(a + b) * x * div_fast(1.0, a + 1.0), 1.0, A1, A2, B1, B2);   // d_1
        wallis_step(de, 1.0, A1, A2, B1, B2);
        const double Ap = A1, Bp = B1;
        wallis_step(d_o, 1.0, A1, A2, B1, B2);
        if (fabs(fma(A1, Bp, -Ap * B1)) <= 1e-16 * fabs(A1 * Bp)) break;
    }
    return div_fast(A1, B1);
}
// log B(m/2, 1/2), the t_1 CDF normaliser; the E-step takes it from CompDev::lbt (per component,
// df m0, m0+1, m0+2) so the per-pair T_1 evaluations carry no lgamma.
__device__ inline double dev_t_lbeta(double m) {
    return lgamma(0.5 * m) + 0.5723649429247001 - lgamma(0.5 * m + 0.5);   // lgamma(1/2) = log(pi)/2
}

// Univariate Student-t CDF with real df m:  P(T <= t) = 1 - I_{m/(m+t^2)}(m/2, 1/2)/2 for t >= 0;
// lbeta = log B(m/2, 1/2) (dev_t_lbeta).
__device__ inline double dev_t_cdf(double t, double m, double lbeta) {
    if (isinf(t)) return t > 0 ? 1.0 : 0.0;
    const double t2 = t * t;
    const double x = m / (m + t2), xc = t2 / (m + t2);
    const double a = 0.5 * m, b = 0.5;
    const double lx = (x > 0.5) ? log1p(-xc) : log(x);
    const double lxc = (xc > 0.5) ? log1p(-x) : log(xc);
    const double front = exp(a * lx + b * lxc - lbeta);
    double tail;   // P(T <= -|t|) = I_x(a, b) / 2
    if (x < (a + 1.0) / (a + b + 2.0)) tail = 0.5 * front * dev_betacf(a, b, x) / a;
    else tail = 0.5 * (1.0 - front * dev_betacf(b, a, xc) / b);
    if (!(xc > 0.0)) tail = 0.5;
    return (t >= 0.0) ? 1.0 - tail : tail;
}
__device__ inline double dev_t_cdf(double t, double m) { return dev_t_cdf(t, m, dev_t_lbeta(m)); }

// log of the univariate t density t_1(0; loc, s2, m) given lgc = lgamma((m+1)/2) - lgamma(m/2).
__device__ __forceinline__ double dev_t1_logpdf0(double loc, double s2, double m, double lgc) {
    return lgc - 0.5 * log(m * CUDART_PI * s2) - 0.5 * (m + 1.0) * log1p(loc * loc / (m * s2));
}

// log of the univariate normal density phi(0; loc, s2) (skew-normal family, reading F1).
__device__ __forceinline__ double dev_n1_logpdf0(double loc, double s2) {
    return -0.5 * loc * loc / s2 - 0.5 * log(2.0 * CUDART_PI * s2);
}

// Regularized incomplete gamma: series for P (x < a + 1), Legendre CF for Q otherwise.
__device__ inline double dev_gamma_series_P(double a, double x, double lga) {
    // branch-free reciprocals (div_fast): x/(a+k) does not depend on the running term, so successive
    // steps overlap instead of serialising on IEEE division's slow-path test
    double sum = div_fast(1.0, a), term = sum, ap = a;
    for (int k = 0; k < 10000; ++k) {
        ap += 1.0;
        term *= div_fast(x, ap);
        sum += term;
        if (fabs(term) <= fabs(sum) * 1e-17) break;
    }
    return sum * exp(a * log(x) - x - lga);
}
// Legendre's continued fraction (DLMF 8.9.2, even form): Gamma(a,x) = e^{-x} x^a cf,
//   cf = 1/(x+1-a - 1(1-a)/(x+3-a - 2(2-a)/(x+5-a - ...))): a_1 = 1, a_n = -(n-1)(n-1-a), b_n = x+2n-1-a.
__device__ inline double dev_gamma_cf_Q(double a, double x, double lga) {
    double A2 = 1.0, B2 = 0.0, A1 = 0.0, B1 = 1.0;
    wallis_step(1.0, x + 1.0 - a, A1, A2, B1, B2);
    for (int n = 2; n < 10000; ++n) {
        const double Ap = A1, Bp = B1;
        wallis_step(-double(n - 1) * (double(n - 1) - a), x + 2.0 * n - 1.0 - a, A1, A2, B1, B2);
        if (fabs(fma(A1, Bp, -Ap * B1)) <= 1e-16 * fabs(A1 * Bp)) break;
    }
    return exp(a * log(x) - x - lga) * div_fast(A1, B1);
}
// log P(a,x) (upper = 0) or log Q(a,x) (upper = 1); lga = lgamma(a) (computed once by the caller)
__device__ inline double dev_log_gamma_PQ(double a, double x, int upper, double lga) {
    if (x < a + 1.0) {
        const double P = dev_gamma_series_P(a, x, lga);
        return upper ? log1p(-P) : log(P);
    }
    const double Q = dev_gamma_cf_Q(a, x, lga);
    return upper ? log(Q) : log1p(-Q);
}

// Chi-square quantile for real df m: solve P(m/2, v/2) = w (w <= 1/2) or Q(m/2, v/2) = 1 - w.
// Newton on log F in s = log(v/2), bracketed; Wilson-Hilferty start.
__device__ inline double dev_chi2_quantile(double w, double m) {
    const double a = 0.5 * m;
    const double lga = lgamma(a);
    const int upper = (w > 0.5);
    const double ltarget = log(upper ? (1.0 - w) : w);
    const double zq = Phiinv(w);
    const double h9 = 2.0 / (9.0 * m);
    double v = m * pow(fmax(1.0 - h9 + zq * sqrt(h9), 1e-3), 3.0);
    double s = log(0.5 * v);
    // small-v regime: P ~ x^a / Gamma(a+1)
    const double s_small = (log(w) + lga + log(a)) / a;   // lgamma(a+1) = lgamma(a) + log(a)
    if (!upper && s_small < s) s = s_small;
    // a-priori bracket, no evaluation: at x = e^{-745} log P ~ -745 a (below any log w), and at
    // x = a e^{40} log Q ~ -x (below any log(1 - w) >= log 2^-53), so the root s lies in (lo, hi)
    double lo = -745.0, hi = fmax(0.0, log(a)) + 40.0;
    if (!(s > lo && s < hi)) s = 0.5 * (lo + hi);
    for (int it = 0; it < 300; ++it) {
        const double x = exp(s);
        const double lF = dev_log_gamma_PQ(a, x, upper, lga);
        const double g = lF - ltarget;
        if (g == 0.0) break;
        const bool root_below = upper ? (g < 0.0) : (g > 0.0);
        if (root_below) hi = s; else lo = s;
        // d log F / ds = x f(x) / F, f the Gamma(a,1) density; negative for Q
        const double ldens = a * log(x) - x - lga;
        double dg = exp(ldens - lF);
        if (upper) dg = -dg;
        double sn = s - g / dg;
        if (fabs(sn - s) <= 1e-12 * fmax(1.0, fabs(s))) { s = sn; break; }
        if (!(sn > lo && sn < hi)) sn = 0.5 * (lo + hi);
        s = sn;
    }
    return 2.0 * exp(s);
}

// ---- 1-D bulk copies (TMA engine) global -> shared with mbarrier completion (sm_90+/sm_100a) ----
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t *m, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(m)), "r"(count) : "memory");
}
// make mbarrier inits and prior generic-proxy shared-memory accesses visible to the async proxy
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(m)), "r"(bytes) : "memory");
}
// bytes: multiple of 16; src and dst 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *m) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, uint32_t parity) {
    asm volatile("{\n\t.reg .pred P1;\n"
                 "WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@!P1 bra WAIT_%=;\n}"
                 ::"r"(smem_addr(m)), "r"(parity) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace cfust
