/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see cfust_oracle.h).
 *
 * Plain FP64 CPU implementation of one FM-CFUST EM iteration, written from the paper
 * (arXiv 2005.06848, /root/reference/PAPER.md) and the readings in DESIGN.md §3 where the
 * paper omits the CFUST E-/M-step ("technical details ... omitted", PAPER.md:194-195;
 * "eight partial sums ... equations (27) to (34) in [llm19]").
 *
 * Notation: r = y - mu, d = r' Omega^{-1} r, c = Delta' Omega^{-1} r,
 * m0 = nu + p, rho = nu + d, S' = (rho/m0) Lambda.  T_r(b; 0, S, m) = P(X <= b),
 * X ~ t_r(0, S, m).  No blocking, fusion or reordering beyond the formulas; per-pair work
 * may run on several threads (independent pairs), the sums are accumulated serially in
 * ascending j.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC cfust_oracle.c -lm
 */
#include "cfust_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define QMAX 8
#define PMAX 8
/* Reading A16: a T_q (or Phi_q) value below the smallest normal double is treated as an
 * underflow, f_ij = 0 — in gradual underflow the ratios E1/T0, E2/T0 lose their precision. */
#define ORC_TMIN 2.2250738585072014e-308
static const double ORC_PI = 3.14159265358979323846;
static const double ORC_UMIN = 1e-300;                 /* reading A15 */
static const double ORC_UMAX = 0x1.fffffffffffffp-1;   /* largest double < 1, reading A15 */

/* =====================================================================================
 * Special functions (pins C12: tests/test_oracle_special.py against scipy / mpmath)
 * ===================================================================================== */

/* Standard normal CDF via the C library erfc: Phi(x) = erfc(-x/sqrt 2)/2. */
double orc_norm_cdf(double x) { return 0.5 * erfc(-x / sqrt(2.0)); }

static double norm_pdf(double x) { return exp(-0.5 * x * x) / sqrt(2.0 * ORC_PI); }

/* Phi^{-1}(u): the root of log Phi(z) = log u, by bisection-safeguarded Newton started from
 * the Abramowitz & Stegun 26.2.23 approximation.  u > 1/2 uses symmetry with 1-u (exact). */
double orc_norm_quantile(double u) {
    if (!(u > 0.0)) return -INFINITY;
    if (!(u < 1.0)) return INFINITY;
    if (u == 0.5) return 0.0;
    if (u > 0.5) return -orc_norm_quantile(1.0 - u);
    const double lu = log(u);
    const double t = sqrt(-2.0 * lu);
    double z = -(t - (2.515517 + 0.802853 * t + 0.010328 * t * t) /
                         (1.0 + 1.432788 * t + 0.189269 * t * t + 0.001308 * t * t * t));
    double lo = -40.0, hi = 0.0;
    for (int it = 0; it < 200; ++it) {
        const double P = orc_norm_cdf(z);
        const double h = log(P) - lu;                 /* increasing in z */
        if (h == 0.0) return z;
        if (h > 0.0) hi = z; else lo = z;
        double zn = z - h * P / norm_pdf(z);          /* Newton on log Phi */
        if (fabs(zn - z) <= 1e-12 * fmax(1.0, fabs(z))) return zn;  /* quadratic: error ~ step^2 */
        if (!(zn > lo && zn < hi)) zn = 0.5 * (lo + hi);
        z = zn;
    }
    return z;
}

/* Regularized incomplete gamma P(a,x) for x < a+1: the series of DLMF 8.7.1,
 *   gamma*(a,x) x^a = e^{-x} x^a / Gamma(a+1) * sum_{k>=0} x^k / ((a+1)(a+2)...(a+k)),
 * summed term by term until a term no longer changes the sum. */
static double gamma_p_series(double a, double x) {
    double sum = 0.0, term = 1.0;
    for (int k = 0; k < 100000; ++k) {
        const double before = sum;
        sum += term;
        if (sum == before) break;
        term = term * x / (a + k + 1.0);
    }
    return exp(a * log(x) - x - lgamma(a + 1.0)) * sum;
}

/* Evaluate the continued fraction  K = a_1/(b_1 + a_2/(b_2 + a_3/(b_3 + ...)))  by the
 * fundamental (Wallis) recurrences A_n = b_n A_{n-1} + a_n A_{n-2}, B_n = b_n B_{n-1} + a_n B_{n-2}
 * (A_{-1} = 1, A_0 = 0, B_{-1} = 0, B_0 = 1), K_n = A_n / B_n, rescaling (A, B) by a power of two
 * whenever |B_n| leaves [2^-500, 2^500] (the ratio is unchanged).  Stops when K_n repeats
 * K_{n-1} to 1e-16 relative.  The coefficient callback gives (a_n, b_n) for n >= 1. */
typedef void (*cf_coef_fn)(int n, const double *par, double *an, double *bn);
static double cf_wallis(cf_coef_fn coef, const double *par) {
    double A2 = 1.0, A1 = 0.0, B2 = 0.0, B1 = 1.0, K = 0.0;
    for (int n = 1; n < 200000; ++n) {
        double an, bn;
        coef(n, par, &an, &bn);
        const double A = bn * A1 + an * A2, B = bn * B1 + an * B2;
        A2 = A1; B2 = B1; A1 = A; B1 = B;
        const double mb = fabs(B1);
        if (mb > 0x1p500 || (mb < 0x1p-500 && mb > 0.0)) {
            const double s = ldexp(1.0, -ilogb(B1));
            A1 *= s; B1 *= s; A2 *= s; B2 *= s;
        }
        if (B1 == 0.0) continue;
        const double Kn = A1 / B1;
        if (n > 1 && fabs(Kn - K) <= 1e-16 * fabs(Kn)) return Kn;
        K = Kn;
    }
    return K;
}

/* Legendre's continued fraction for the upper incomplete gamma (DLMF 8.9.2 in its even form):
 *   Gamma(a,x) = e^{-x} x^a * 1/(x+1-a - 1(1-a)/(x+3-a - 2(2-a)/(x+5-a - ...))),
 * i.e. a_1 = 1, a_n = -(n-1)(n-1-a) (n >= 2), b_n = x + 2n - 1 - a.  Used for x >= a+1. */
static void gamma_q_coef(int n, const double *par, double *an, double *bn) {
    const double a = par[0], x = par[1];
    *an = (n == 1) ? 1.0 : -(double)(n - 1) * ((double)(n - 1) - a);
    *bn = x + 2.0 * n - 1.0 - a;
}
static double gamma_q_cf(double a, double x) {
    const double par[2] = {a, x};
    return exp(a * log(x) - x - lgamma(a)) * cf_wallis(gamma_q_coef, par);
}

double orc_gamma_p(double a, double x) {
    if (!(x > 0.0)) return 0.0;
    if (isinf(x)) return 1.0;
    return (x < a + 1.0) ? gamma_p_series(a, x) : 1.0 - gamma_q_cf(a, x);
}

double orc_gamma_q(double a, double x) {
    if (!(x > 0.0)) return 1.0;
    if (isinf(x)) return 0.0;
    return (x < a + 1.0) ? 1.0 - gamma_p_series(a, x) : gamma_q_cf(a, x);
}

/* Chi-square quantile with real df m: v such that P(m/2, v/2) = w.  For w > 1/2 the
 * equivalent equation Q(m/2, v/2) = 1-w (1-w exact) is solved.  Newton in t = log(v/2) on
 * log F, safeguarded by bisection in t.  Started from the Wilson-Hilferty approximation. */
double orc_chi2_quantile(double w, double m) {
    if (!(w > 0.0)) return 0.0;
    if (!(w < 1.0)) return INFINITY;
    const double a = 0.5 * m;
    const int upper = w > 0.5;
    const double lt = log(upper ? 1.0 - w : w);
    /* initial guess */
    const double zq = orc_norm_quantile(w);
    const double k9 = 2.0 / (9.0 * m);
    double v0 = m * pow(1.0 - k9 + zq * sqrt(k9), 3.0);
    if (!(v0 > 0.0)) v0 = 2.0 * exp((log(w) + lgamma(a + 1.0)) / a);   /* P ~ x^a / Gamma(a+1) */
    double t = log(0.5 * v0);
    double tlo = -745.0, thi = log(fmax(1.0, a)) ;
    /* expand upper bracket until F(e^thi) is past the target */
    for (int it = 0; it < 200; ++it) {
        const double x = exp(thi);
        const double F = upper ? orc_gamma_q(a, x) : orc_gamma_p(a, x);
        const double h = log(F) - lt;
        if (upper ? (h < 0.0) : (h > 0.0)) break;
        thi += 1.0;
    }
    if (!(t > tlo && t < thi)) t = 0.5 * (tlo + thi);
    for (int it = 0; it < 400; ++it) {
        const double x = exp(t);
        const double F = upper ? orc_gamma_q(a, x) : orc_gamma_p(a, x);
        const double h = log(F) - lt;   /* increasing in t for P, decreasing for Q */
        if (h == 0.0) break;
        if ((h > 0.0) != upper) thi = t; else tlo = t;
        /* d log F / dt = x * pdf(x) / F (sign - for Q) */
        const double lpdf = (a - 1.0) * log(x) - x - lgamma(a);
        double dh = exp(log(x) + lpdf) / F;
        if (upper) dh = -dh;
        double tn = t - h / dh;
        if (fabs(tn - t) <= 1e-12 * fmax(1.0, fabs(t))) { t = tn; break; }  /* quadratic */
        if (!(tn > tlo && tn < thi)) tn = 0.5 * (tlo + thi);
        t = tn;
    }
    return 2.0 * exp(t);
}

/* Continued fraction of the incomplete beta function (DLMF 8.17.22):
 *   I_x(a,b) = x^a (1-x)^b / (a B(a,b)) * 1/(1 + d_1/(1 + d_2/(1 + ...))),
 *   d_{2m} = m(b-m)x / ((a+2m-1)(a+2m)),  d_{2m+1} = -(a+m)(a+b+m)x / ((a+2m)(a+2m+1)),
 * converging quickly for x < (a+1)/(a+b+2).  In the a_n/b_n form: a_1 = 1, a_n = d_{n-1}, b_n = 1. */
static void ibeta_coef(int n, const double *par, double *an, double *bn) {
    const double a = par[0], b = par[1], x = par[2];
    *bn = 1.0;
    if (n == 1) { *an = 1.0; return; }
    const int k = n - 1;              /* d_k */
    if (k % 2 == 0) {
        const double m = 0.5 * k;
        *an = m * (b - m) * x / ((a + k - 1.0) * (a + k));
    } else {
        const double m = 0.5 * (k - 1);
        *an = -(a + m) * (a + b + m) * x / ((a + 2.0 * m) * (a + 2.0 * m + 1.0));
    }
}
static double betacf(double a, double b, double x) {
    const double par[3] = {a, b, x};
    return cf_wallis(ibeta_coef, par);
}

/* Regularized incomplete beta I_x(a,b); xc = 1-x supplied separately for accuracy. */
double orc_ibeta(double a, double b, double x, double xc) {
    if (!(x > 0.0)) return 0.0;
    if (!(xc > 0.0)) return 1.0;
    const double lx = (x < 0.5) ? log(x) : log1p(-xc);
    const double lxc = (xc < 0.5) ? log(xc) : log1p(-x);
    const double lfront = a * lx + b * lxc - (lgamma(a) + lgamma(b) - lgamma(a + b));
    if (x < (a + 1.0) / (a + b + 2.0)) return exp(lfront) * betacf(a, b, x) / a;
    return 1.0 - exp(lfront) * betacf(b, a, xc) / b;
}

/* Univariate Student-t CDF with real df m: T_m(x) = 1 - I_{m/(m+x^2)}(m/2, 1/2)/2 for x >= 0. */
double orc_t_cdf(double x, double m) {
    if (isnan(x)) return NAN;
    if (isinf(x)) return x > 0 ? 1.0 : 0.0;
    const double x2 = x * x;
    const double tail = 0.5 * orc_ibeta(0.5 * m, 0.5, m / (m + x2), x2 / (m + x2));
    return x >= 0.0 ? 1.0 - tail : tail;
}

/* log t_1(x; loc, s2, m): univariate t density with location loc, scale^2 s2, df m. */
double orc_t1_logpdf(double x, double loc, double s2, double m) {
    const double u = (x - loc) * (x - loc) / (m * s2);
    return lgamma(0.5 * (m + 1.0)) - lgamma(0.5 * m) - 0.5 * log(m * ORC_PI * s2)
           - 0.5 * (m + 1.0) * log1p(u);
}

/* Digamma: recurrence psi(x) = psi(x+1) - 1/x up to x >= 10, then the asymptotic series. */
double orc_digamma(double x) {
    double r = 0.0;
    while (x < 10.0) { r -= 1.0 / x; x += 1.0; }
    const double f = 1.0 / (x * x);
    const double t = f * (-1.0 / 12 + f * (1.0 / 120 + f * (-1.0 / 252 + f * (1.0 / 240 +
                     f * (-1.0 / 132 + f * (691.0 / 32760 + f * (-1.0 / 12)))))));
    return r + log(x) - 0.5 / x + t;
}

/* =====================================================================================
 * Small dense linear algebra (row-major)
 * ===================================================================================== */
static int chol(int n, const double *S, double *L) {
    memset(L, 0, sizeof(double) * n * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = S[i * n + j];
            for (int k = 0; k < j; ++k) s -= L[i * n + k] * L[j * n + k];
            if (i == j) {
                if (!(s > 1e-300)) return ORC_ENOTPD;   /* SPEC.md:125 pivot rule */
                L[i * n + i] = sqrt(s);
            } else {
                L[i * n + j] = s / L[j * n + j];
            }
        }
    return ORC_OK;
}

/* solve L L' x = b in place */
static void chol_solve(int n, const double *L, double *x) {
    for (int i = 0; i < n; ++i) {
        double s = x[i];
        for (int k = 0; k < i; ++k) s -= L[i * n + k] * x[k];
        x[i] = s / L[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int k = i + 1; k < n; ++k) s -= L[k * n + i] * x[k];
        x[i] = s / L[i * n + i];
    }
}

int orc_k_stats(int p, int q) { return 3 + p + p * (p + 1) / 2 + q + q * (q + 1) / 2 + p * q; }

/* =====================================================================================
 * Lattice (O0; readings A11, A12): x = frac((l z_k mod M)/M + shift_k), w = |2x - 1|.
 * ===================================================================================== */
double orc_lattice_w(const orc_lattice *L, int64_t l, int k) {
    const uint64_t t = ((uint64_t)l * (uint64_t)L->z[k]) % (uint64_t)L->M;
    double x = (double)t / (double)L->M + L->shift[k];
    if (x >= 1.0) x -= 1.0;
    return fabs(2.0 * x - 1.0);
}

/* Chi radius nodes for df m: s_l = sqrt(chi2_m^{-1}(w_{l,0}) / m)  (reading R-T). */
void orc_chi_table(const orc_lattice *L, double m, double *s_out) {
    for (int64_t l = 0; l < L->M; ++l) s_out[l] = sqrt(orc_chi2_quantile(orc_lattice_w(L, l, 0), m) / m);
}

/* log V_l = log chi2_m^{-1}(w_{l,0}): the log of the chi-square node behind s_l (exact e1, R2'). */
void orc_logchi_table(const orc_lattice *L, double m, double *out) {
    for (int64_t l = 0; l < L->M; ++l) out[l] = log(orc_chi2_quantile(orc_lattice_w(L, l, 0), m));
}

/* Reading A14 (test harness): keys within 1e-12 max(1, |key|) of each other are near-ties, for which
 * several variable orders are valid.  orc_set_tie_flip(1) sorts every near-tied pair in the opposite
 * order (the later variable first), so the parity tests can accept a GPU result that matches the
 * oracle under either order; the default (0) is the stable ascending order of reading A13. */
static int g_tie_flip = 0;
void orc_set_tie_flip(int on) { g_tie_flip = on ? 1 : 0; }
static int key_before(double kj, double ki) {   /* insertion sort: move kj past ki? */
    if (kj > ki) return 1;
    return g_tie_flip && fabs(kj - ki) <= 1e-12 * fmax(1.0, fmax(fabs(kj), fabs(ki)));
}

/* =====================================================================================
 * T_r(b; 0, S, m) — Genz-Bretz separation of variables for the multivariate t in its
 * chi-normal form (reading R-T):  T_r(b;S,m) = E_V[ Phi_r( b sqrt(V/m); S ) ],
 * V ~ chi^2_m.  Lattice coordinate 0 gives V, coordinates 1..r-1 the normal SOV steps.
 * Variables are reordered by ascending b_k/sqrt(S_kk), stable (reading A13/A14).
 * r = 0 -> 1;  r = 1 -> closed form T_m(b/sqrt(S)).
 * ===================================================================================== */
/* With lv != NULL (exact e1, reading R2'): also *wsum = (1/M) sum_l f_l lv_l over the same
 * lattice points, and r = 1 is evaluated on the lattice too (f_l = Phi(s_l b / sqrt(S))). */
static double tr_core(int r, const double *b, const double *S, double m, const orc_lattice *L,
                      const double *chi_s, const double *lv, double *min_key_gap, double *wsum) {
    if (r == 0) return 1.0;
    if (r == 1 && lv) {
        double sum = 0.0, ws = 0.0;
        const double bs = b[0] / sqrt(S[0]);
        for (int64_t l = 0; l < L->M; ++l) {
            const double f = orc_norm_cdf(chi_s[l] * bs);
            sum += f;
            ws += f * lv[l];
        }
        *wsum = ws / (double)L->M;
        return sum / (double)L->M;
    }
    if (r == 1) return orc_t_cdf(b[0] / sqrt(S[0]), m);
    int perm[QMAX];
    double key[QMAX];
    for (int k = 0; k < r; ++k) { perm[k] = k; key[k] = b[k] / sqrt(S[k * r + k]); }
    for (int i = 1; i < r; ++i) {   /* stable insertion sort by key */
        const int pi = perm[i];
        int j = i - 1;
        while (j >= 0 && key_before(key[perm[j]], key[pi])) { perm[j + 1] = perm[j]; --j; }
        perm[j + 1] = pi;
    }
    if (min_key_gap) {
        for (int i = 1; i < r; ++i) {
            const double a = key[perm[i - 1]], bb = key[perm[i]];
            const double gap = fabs(bb - a) / fmax(1.0, fmax(fabs(a), fabs(bb)));
            if (gap < *min_key_gap) *min_key_gap = gap;
        }
    }
    double Sp[QMAX * QMAX], bp[QMAX], C[QMAX * QMAX];
    for (int i = 0; i < r; ++i) {
        bp[i] = b[perm[i]];
        for (int j = 0; j < r; ++j) Sp[i * r + j] = S[perm[i] * r + perm[j]];
    }
    if (chol(r, Sp, C) != ORC_OK) return NAN;
    double sum = 0.0, ws = 0.0;
    for (int64_t l = 0; l < L->M; ++l) {
        const double s = chi_s[l];
        double e = orc_norm_cdf(s * bp[0] / C[0]);
        double f = e;
        double zz[QMAX];
        for (int k = 1; k < r; ++k) {
            double u = orc_lattice_w(L, l, k) * e;
            if (u < ORC_UMIN) u = ORC_UMIN;
            if (u > ORC_UMAX) u = ORC_UMAX;
            zz[k - 1] = orc_norm_quantile(u);
            double acc = s * bp[k];
            for (int t = 0; t < k; ++t) acc -= C[k * r + t] * zz[t];
            e = orc_norm_cdf(acc / C[k * r + k]);
            f *= e;
        }
        sum += f;
        if (lv) ws += f * lv[l];
    }
    if (lv) *wsum = ws / (double)L->M;
    return sum / (double)L->M;
}

double orc_Tr(int r, const double *b, const double *S, double m, const orc_lattice *L,
              const double *chi_s, double *min_key_gap) {
    return tr_core(r, b, S, m, L, chi_s, NULL, min_key_gap, NULL);
}

double orc_Tr_w(int r, const double *b, const double *S, double m, const orc_lattice *L,
                const double *chi_s, const double *lv, double *min_key_gap, double *wsum) {
    return tr_core(r, b, S, m, L, chi_s, lv, min_key_gap, wsum);
}

/* =====================================================================================
 * O1: per-component derived quantities (Eq. (2) definitions)
 *   Omega = Sigma + Delta Delta', L_omega = chol(Omega), A = Delta' Omega^{-1} (q x p),
 *   Lambda = I_q - Delta' Omega^{-1} Delta (symmetrised),
 *   kappa = lgamma((nu+p)/2) - lgamma(nu/2) - (p/2) log(nu pi) - (1/2) log|Omega|.
 * ===================================================================================== */
int orc_derive(int p, int q, const double *sigma, const double *delta, double nu,
               double *L_omega, double *A, double *Lambda, double *logdet, double *kappa) {
    double Om[PMAX * PMAX];
    for (int a = 0; a < p; ++a)
        for (int b = 0; b < p; ++b) {
            double s = sigma[a * p + b];
            for (int k = 0; k < q; ++k) s += delta[a * q + k] * delta[b * q + k];
            Om[a * p + b] = s;
        }
    if (chol(p, Om, L_omega) != ORC_OK) return ORC_ENOTPD;
    double ld = 0.0;
    for (int a = 0; a < p; ++a) ld += 2.0 * log(L_omega[a * p + a]);
    *logdet = ld;
    for (int k = 0; k < q; ++k) {          /* column k of Omega^{-1} Delta */
        double x[PMAX];
        for (int a = 0; a < p; ++a) x[a] = delta[a * q + k];
        chol_solve(p, L_omega, x);
        for (int a = 0; a < p; ++a) A[k * p + a] = x[a];
    }
    for (int k = 0; k < q; ++k)
        for (int l = 0; l < q; ++l) {
            double s = 0.0;
            for (int a = 0; a < p; ++a) s += delta[a * q + k] * A[l * p + a];
            Lambda[k * q + l] = (k == l ? 1.0 : 0.0) - s;
        }
    for (int k = 0; k < q; ++k)
        for (int l = k + 1; l < q; ++l) {
            const double s = 0.5 * (Lambda[k * q + l] + Lambda[l * q + k]);
            Lambda[k * q + l] = Lambda[l * q + k] = s;
        }
    const double m0 = nu + p;
    *kappa = lgamma(0.5 * m0) - lgamma(0.5 * nu) - 0.5 * p * log(nu * ORC_PI) - 0.5 * ld;
    return ORC_OK;
}

/* Parity-harness output (tests only; no effect on the E-step): running error bounds of the two
 * cancelling sums of O7, in the units of e3 / e4.  E1 = c T2 + S'h and E2 = sym(S'(G + T0 I) + c E1')
 * are sums of terms of either sign; if every integral (T2, T~(k), T(k,t)) and density factor carries a
 * relative perturbation <= delta, each moment moves by at most delta times the same sum taken over
 * |terms|:  B1_a = |c_a T2| + sum_k |S'_ak h_k|,  B2_ab = sum_k |S'_ak| (BG_kb + [k = b] T0) + |c_a| B1_b
 * (BG_kb = |phi_k| (|c~_b T~(k)| + sum |S~'(k) h(k)|)).  bound[0..q) = (m0/rho) B1 / T0,
 * bound[q + a q + b] = (m0/rho) (B2_ab + B2_ba) / (2 T0).  In the deep tail of a component
 * (alpha = c / sqrt(S') << 0) B / |moment| grows like alpha^2 (E1) and alpha^4 (E2): the condition
 * number of the formula (reading P1). */
static void moment_bounds(int q, const double *c, const double *Sp, const double *h, double T2, double T0,
                          const double *BG, double fac, double *bound) {
    double B1[QMAX];
    for (int a = 0; a < q; ++a) {
        double s = fabs(c[a] * T2);
        for (int k = 0; k < q; ++k) s += fabs(Sp[a * q + k] * h[k]);
        B1[a] = s;
        bound[a] = fac * s / T0;
    }
    double B2[QMAX * QMAX];
    for (int a = 0; a < q; ++a)
        for (int b = 0; b < q; ++b) {
            double s = 0.0;
            for (int k = 0; k < q; ++k) s += fabs(Sp[a * q + k]) * (BG[k * q + b] + (k == b ? T0 : 0.0));
            B2[a * q + b] = s + fabs(c[a]) * B1[b];
        }
    for (int a = 0; a < q; ++a)
        for (int b = 0; b < q; ++b) bound[q + a * q + b] = fac * 0.5 * (B2[a * q + b] + B2[b * q + a]) / T0;
}

/* =====================================================================================
 * O2-O8: one (observation, component) pair.
 * out = [log(2^q t_p T0)  (no log pi),  e1-e2,  e2,  e3 (q),  e4 (q*q)]
 * e1 = E[log W | y]: lv_m0 == NULL -> the closed-form approximation (reading A5, R1);
 * lv_m0 = log chi2_{m0}^{-1} node table -> exact (reading R2'):  with V ~ chi2_{m0} and
 * W = V / rho a posteriori weighted by Phi_q(c sqrt(V/rho); Lambda),
 *   e1 = E_V[log(V/rho) Phi_q] / E_V[Phi_q] = (sum_l f_l log V_l) / (sum_l f_l) - log rho
 * on T0's own lattice points (f_l the SOV integrand of T0).
 * ===================================================================================== */
int orc_pair(int p, int q, const double *y, const double *mu, const double *L_omega,
             const double *A, const double *Lambda, double nu, double kappa,
             const orc_lattice *L, const double *chi_m0, const double *chi_m1,
             const double *chi_m2, const double *lv_m0, double *out, double *min_key_gap, double *bound) {
    double r[PMAX], v[PMAX];
    for (int a = 0; a < p; ++a) r[a] = y[a] - mu[a];
    for (int a = 0; a < p; ++a) {          /* forward solve L v = r; d = |v|^2 */
        double s = r[a];
        for (int b = 0; b < a; ++b) s -= L_omega[a * p + b] * v[b];
        v[a] = s / L_omega[a * p + a];
    }
    double d = 0.0;
    for (int a = 0; a < p; ++a) d += v[a] * v[a];
    const double m0 = nu + p, rho = nu + d;
    const double logt = kappa - 0.5 * m0 * log1p(d / nu);              /* log t_p(y; mu, Omega, nu) */
    const double e1me2 = orc_digamma(0.5 * m0) - log(0.5 * rho) - m0 / rho;   /* reading A5 (R1) */
    out[1] = e1me2;
    if (q == 0) {                            /* Delta = 0: t-mixture */
        out[0] = logt;
        out[2] = m0 / rho;
        return ORC_OK;
    }
    double c[QMAX];
    for (int k = 0; k < q; ++k) {
        double s = 0.0;
        for (int a = 0; a < p; ++a) s += A[k * p + a] * r[a];
        c[k] = s;
    }
    /* T0 for the density (Eq. (2)), T2 for e2 */
    double bq[QMAX];
    for (int k = 0; k < q; ++k) bq[k] = c[k] * sqrt(m0 / rho);
    double e1_exact = 0.0;
    double T0;
    if (lv_m0) {
        double wsum = 0.0;
        const double T0lat = orc_Tr_w(q, bq, Lambda, m0, L, chi_m0, lv_m0, min_key_gap, &wsum);
        T0 = (q == 1) ? orc_Tr(1, bq, Lambda, m0, L, chi_m0, NULL) : T0lat;   /* density: exact T_1 */
        e1_exact = wsum / T0lat - log(rho);
    } else {
        T0 = orc_Tr(q, bq, Lambda, m0, L, chi_m0, min_key_gap);
    }
    for (int k = 0; k < q; ++k) bq[k] = c[k] * sqrt((m0 + 2.0) / rho);
    const double T2 = orc_Tr(q, bq, Lambda, m0 + 2.0, L, chi_m2, min_key_gap);
    const int PW = 3 + q + q * q;
    if (!(T0 >= ORC_TMIN)) {                 /* reading A16: f_ij = 0 (T0 below the normal FP64 range) */
        out[0] = -INFINITY;
        for (int k = 2; k < PW; ++k) out[k] = 0.0;
        return ORC_OK;
    }
    double Sp[QMAX * QMAX];                  /* S' = (rho/m0) Lambda */
    for (int k = 0; k < q * q; ++k) Sp[k] = (rho / m0) * Lambda[k];

    /* O6: h_k = t_1(0; c_k, S'_kk, m0) * T_{q-1}(c~(k); 0, S~(k), m0+1) */
    const int q1 = q - 1;
    double phi[QMAX], Tk[QMAX], h[QMAX];
    double ct[QMAX][QMAX], St[QMAX][QMAX * QMAX], Stp[QMAX][QMAX * QMAX];
    int oth[QMAX][QMAX];
    for (int k = 0; k < q; ++k) {
        phi[k] = exp(orc_t1_logpdf(0.0, c[k], Sp[k * q + k], m0));
        Tk[k] = 1.0;
        if (q >= 2) {
            int na = 0;
            for (int t = 0; t < q; ++t) if (t != k) oth[k][na++] = t;
            const double skk = Sp[k * q + k];
            const double fac = (m0 + c[k] * c[k] / skk) / (m0 + 1.0);
            for (int a = 0; a < q1; ++a) {
                const int ia = oth[k][a];
                ct[k][a] = c[ia] - Sp[ia * q + k] * c[k] / skk;
                for (int b = 0; b < q1; ++b) {
                    const int ib = oth[k][b];
                    St[k][a * q1 + b] = fac * (Sp[ia * q + ib] - Sp[ia * q + k] * Sp[k * q + ib] / skk);
                }
            }
            Tk[k] = orc_Tr(q1, ct[k], St[k], m0 + 1.0, L, chi_m1, min_key_gap);
            for (int a = 0; a < q1 * q1; ++a) Stp[k][a] = ((m0 + 1.0) / (m0 - 1.0)) * St[k][a];
        }
        h[k] = phi[k] * Tk[k];
    }
    /* O7: E1 = E[X 1{X>0}], X ~ t_q(c, S, m0+2):  E1 = c T2 + S' h */
    double E1[QMAX];
    for (int a = 0; a < q; ++a) {
        double s = c[a] * T2;
        for (int k = 0; k < q; ++k) s += Sp[a * q + k] * h[k];
        E1[a] = s;
    }
    /* G_kl = phi_k * E[X_l 1{X_-k > 0} | X_k = 0] (first moment of the conditional truncated t):
     *      = phi_k [ c~(k)_l T~(k) + (S~'(k) h(k))_l ],  G_kk = 0,
     * h(k)_t = t_1(0; c~(k)_t, S~'(k)_tt, m0-1) * T_{q-2}(c^(k,t); 0, S^(k,t), m0). */
    double G[QMAX * QMAX], BG[QMAX * QMAX];   /* BG: running bound sum |terms| of G (test output) */
    memset(G, 0, sizeof(G));
    memset(BG, 0, sizeof(BG));
    if (q >= 2) {
        const int q2 = q - 2;
        double Tkt[QMAX][QMAX];
        for (int k = 0; k < q; ++k)
            for (int t = k + 1; t < q; ++t) {
                double val = 1.0;
                if (q2 >= 1) {
                    int at = -1;
                    for (int a = 0; a < q1; ++a) if (oth[k][a] == t) at = a;
                    const double saa = Stp[k][at * q1 + at];
                    const double fac2 = (m0 - 1.0 + ct[k][at] * ct[k][at] / saa) / m0;
                    double ch[QMAX], Sh[QMAX * QMAX];
                    int rest[QMAX], nr = 0;
                    for (int a = 0; a < q1; ++a) if (a != at) rest[nr++] = a;
                    for (int a = 0; a < q2; ++a) {
                        const int ra = rest[a];
                        ch[a] = ct[k][ra] - Stp[k][ra * q1 + at] * ct[k][at] / saa;
                        for (int b = 0; b < q2; ++b) {
                            const int rb = rest[b];
                            Sh[a * q2 + b] = fac2 * (Stp[k][ra * q1 + rb] -
                                                     Stp[k][ra * q1 + at] * Stp[k][at * q1 + rb] / saa);
                        }
                    }
                    val = orc_Tr(q2, ch, Sh, m0, L, chi_m0, min_key_gap);
                }
                Tkt[k][t] = Tkt[t][k] = val;   /* symmetric in {k,t}: evaluated once (A17) */
            }
        for (int k = 0; k < q; ++k) {
            double hk[QMAX];
            for (int a = 0; a < q1; ++a) {
                const int t = oth[k][a];
                hk[a] = exp(orc_t1_logpdf(0.0, ct[k][a], Stp[k][a * q1 + a], m0 - 1.0)) * Tkt[k][t];
            }
            for (int a = 0; a < q1; ++a) {
                double s = ct[k][a] * Tk[k];
                for (int b = 0; b < q1; ++b) s += Stp[k][a * q1 + b] * hk[b];
                G[k * q + oth[k][a]] = phi[k] * s;
                if (bound) {
                    double sb = fabs(ct[k][a] * Tk[k]);
                    for (int b = 0; b < q1; ++b) sb += fabs(Stp[k][a * q1 + b] * hk[b]);
                    BG[k * q + oth[k][a]] = fabs(phi[k]) * sb;
                }
            }
        }
    }
    /* E2 = E[X X' 1{X>0}] = sym( S'(G + T0 I) + c E1' ) */
    double E2[QMAX * QMAX];
    for (int a = 0; a < q; ++a)
        for (int b = 0; b < q; ++b) {
            double s = 0.0;
            for (int k = 0; k < q; ++k) s += Sp[a * q + k] * (G[k * q + b] + (k == b ? T0 : 0.0));
            E2[a * q + b] = s + c[a] * E1[b];
        }
    /* O8 */
    const double fac = m0 / rho;
    out[0] = q * log(2.0) + logt + log(T0);
    out[2] = fac * T2 / T0;
    if (lv_m0) out[1] = e1_exact - out[2];
    for (int a = 0; a < q; ++a) out[3 + a] = fac * E1[a] / T0;
    for (int a = 0; a < q; ++a)
        for (int b = 0; b < q; ++b)
            out[3 + q + a * q + b] = fac * 0.5 * (E2[a * q + b] + E2[b * q + a]) / T0;
    if (bound) moment_bounds(q, c, Sp, h, T2, T0, BG, fac, bound);
    return ORC_OK;
}

/* =====================================================================================
 * SOV-direct truncated-moment estimator (NEXT-3, reading D1; flag ORC_DIRECT).  Instead of the
 * analytic reduction of O6-O7 to T_{q-1} / T_{q-2} integrals, the moments are estimated on the
 * SOV points of T0 itself, drawing the last normal coordinate too (lattice coordinate q):
 *   per point l: s_l = chi node (df m0), w_l = V_l / rho = m0 s_l^2 / rho, b = s_l c sqrt(m0/rho)
 *   (permuted as T0, ascending c_k / sqrt(Lambda_kk)), e_k and xi_k = Phi^{-1}(u_{l,k+1} e_k) for
 *   k = 0..q-1, z = C xi (C = chol of the permuted Lambda; Z ~ N(0, Lambda) restricted to Z <= b),
 *   U = c - z / sqrt(w_l) (the posterior draw of U given W = w_l), f_l = prod_k e_k;
 *   T0 = (1/M) sum f_l (bit-identical to O4's T0), e2 = sum f w / sum f, e1 = sum f log w / sum f
 *   (exact, as R2'), e3 = sum f w U / sum f, e4 = sum f w U U' / sum f.
 * Skew-normal family: w = 1, s_l = 1.  q = 1: the density keeps the exact T_1.
 * ===================================================================================== */
int orc_pair_direct(int p, int q, const double *y, const double *mu, const double *L_omega,
                    const double *A, const double *Lambda, double nu, double kappa, double logdet, int sn,
                    const orc_lattice *L, const double *chi_m0, const double *lv_m0, double *out,
                    double *min_key_gap) {
    double r[PMAX], v[PMAX];
    for (int a = 0; a < p; ++a) r[a] = y[a] - mu[a];
    for (int a = 0; a < p; ++a) {
        double t = r[a];
        for (int b = 0; b < a; ++b) t -= L_omega[a * p + b] * v[b];
        v[a] = t / L_omega[a * p + a];
    }
    double d = 0.0;
    for (int a = 0; a < p; ++a) d += v[a] * v[a];
    const double m0 = nu + p, rho = nu + d;
    const double logt = sn ? -0.5 * p * log(2.0 * ORC_PI) - 0.5 * logdet - 0.5 * d
                           : kappa - 0.5 * m0 * log1p(d / nu);
    const int PW = 3 + q + q * q;
    if (q == 0) {
        out[0] = logt;
        out[1] = sn ? 0.0 : orc_digamma(0.5 * m0) - log(0.5 * rho) - m0 / rho;
        out[2] = sn ? 1.0 : m0 / rho;
        return ORC_OK;
    }
    double c[QMAX];
    for (int k = 0; k < q; ++k) {
        double t = 0.0;
        for (int a = 0; a < p; ++a) t += A[k * p + a] * r[a];
        c[k] = t;
    }
    const double sq = sn ? 1.0 : sqrt(m0 / rho);
    double bq[QMAX];
    for (int k = 0; k < q; ++k) bq[k] = c[k] * sq;
    int perm[QMAX];
    double key[QMAX];
    for (int k = 0; k < q; ++k) { perm[k] = k; key[k] = bq[k] / sqrt(Lambda[k * q + k]); }
    for (int i = 1; i < q; ++i) {
        const int pi = perm[i];
        int j = i - 1;
        while (j >= 0 && key_before(key[perm[j]], key[pi])) { perm[j + 1] = perm[j]; --j; }
        perm[j + 1] = pi;
    }
    if (min_key_gap)
        for (int i = 1; i < q; ++i) {
            const double a = key[perm[i - 1]], bb = key[perm[i]];
            const double gap = fabs(bb - a) / fmax(1.0, fmax(fabs(a), fabs(bb)));
            if (gap < *min_key_gap) *min_key_gap = gap;
        }
    double Sp[QMAX * QMAX], bp[QMAX], cp[QMAX], C[QMAX * QMAX];
    for (int i = 0; i < q; ++i) {
        bp[i] = bq[perm[i]];
        cp[i] = c[perm[i]];
        for (int j = 0; j < q; ++j) Sp[i * q + j] = Lambda[perm[i] * q + perm[j]];
    }
    if (chol(q, Sp, C) != ORC_OK) return ORC_ENOTPD;
    double F = 0.0, FW = 0.0, FL = 0.0, F3[QMAX] = {0}, F4[QMAX * QMAX] = {0};
    const double lrho = log(rho);
    for (int64_t l = 0; l < L->M; ++l) {
        const double s = chi_m0[l];
        double e = orc_norm_cdf(s * bp[0] / C[0]);
        double f = e;
        double xi[QMAX];
        for (int k = 0; k < q; ++k) {
            if (k > 0) {
                double acc = s * bp[k];
                for (int t = 0; t < k; ++t) acc -= C[k * q + t] * xi[t];
                e = orc_norm_cdf(acc / C[k * q + k]);
                f *= e;
            }
            double u = orc_lattice_w(L, l, k + 1) * e;
            if (u < ORC_UMIN) u = ORC_UMIN;
            if (u > ORC_UMAX) u = ORC_UMAX;
            xi[k] = orc_norm_quantile(u);
        }
        const double w = sn ? 1.0 : m0 * s * s / rho;
        const double sw = sn ? 1.0 : s * sq;                  /* sqrt(w) */
        double U[QMAX];
        for (int k = 0; k < q; ++k) {
            double z = 0.0;
            for (int t = 0; t <= k; ++t) z += C[k * q + t] * xi[t];
            U[perm[k]] = cp[k] - z / sw;
        }
        F += f;
        FW += f * w;
        if (!sn) FL += f * (lv_m0[l] - lrho);
        for (int a = 0; a < q; ++a) {
            F3[a] += f * w * U[a];
            for (int b = a; b < q; ++b) F4[a * q + b] += f * w * U[a] * U[b];
        }
    }
    const double T0lat = F / (double)L->M;
    const double T0 = (q == 1) ? (sn ? orc_norm_cdf(bq[0] / sqrt(Lambda[0])) : orc_t_cdf(bq[0] / sqrt(Lambda[0]), m0))
                               : T0lat;
    if (!(T0 >= ORC_TMIN) || !(F > 0.0)) {                /* reading A16 */
        out[0] = -INFINITY;
        out[1] = sn ? 0.0 : orc_digamma(0.5 * m0) - log(0.5 * rho) - m0 / rho;
        for (int k = 2; k < PW; ++k) out[k] = 0.0;
        return ORC_OK;
    }
    out[0] = q * log(2.0) + logt + log(T0);
    out[2] = FW / F;
    out[1] = sn ? 0.0 : FL / F - out[2];
    for (int a = 0; a < q; ++a) out[3 + a] = F3[a] / F;
    for (int a = 0; a < q; ++a)
        for (int b = a; b < q; ++b) out[3 + q + a * q + b] = out[3 + q + b * q + a] = F4[a * q + b] / F;
    return ORC_OK;
}

/* =====================================================================================
 * Skew-normal family (CFUSN, NEXT-3): the nu -> infinity limit of Eq. (2) (
 * reading F1).  W = 1, so U | y ~ N_q(c, Lambda) restricted to u > 0 and
 *   f = 2^q phi_p(y; mu, Omega) Phi_q(c; 0, Lambda),  e2 = 1,  e3 = E1 / P,  e4 = E2 / P,
 * with the truncated-normal moments of X ~ N_q(c, Lambda) on X > 0 (Tallis):
 *   P = Phi_q(c; Lambda),  E1 = c P + Lambda h,  h_k = phi(0; c_k, Lambda_kk) Phi_{q-1}(c~(k); S~(k)),
 *   E2 = sym( Lambda (G + P I) + c E1' ),  G_kl = phi_k [ c~(k)_l P~(k) + (S~(k) h(k))_l ],
 *   h(k)_t = phi(0; c~(k)_t, S~(k)_tt) Phi_{q-2}(c^(k,t); S^(k,t)),
 * (c~(k), S~(k)) the normal conditional on x_k = 0.  Phi_r is the chi-normal lattice rule of
 * orc_Tr with every radius node s_l = 1 (the normal SOV on the same lattice coordinates 1..r-1);
 * Phi_1 is erfc-exact.  out = [log(2^q phi_p P), 0 (no e1 - e2), 1 (e2), e3 (q), e4 (q*q)].
 * ===================================================================================== */
static double norm_logpdf0(double loc, double s2) { return -0.5 * loc * loc / s2 - 0.5 * log(2.0 * ORC_PI * s2); }

static double phi_r(int r, const double *b, const double *S, const orc_lattice *L, const double *ones,
                    double *min_key_gap) {
    if (r == 0) return 1.0;
    if (r == 1) return orc_norm_cdf(b[0] / sqrt(S[0]));
    return tr_core(r, b, S, INFINITY, L, ones, NULL, min_key_gap, NULL);
}

int orc_pair_sn(int p, int q, const double *y, const double *mu, const double *L_omega,
                const double *A, const double *Lambda, double logdet, const orc_lattice *L,
                const double *ones, double *out, double *min_key_gap, double *bound) {
    double r[PMAX], v[PMAX];
    for (int a = 0; a < p; ++a) r[a] = y[a] - mu[a];
    for (int a = 0; a < p; ++a) {
        double s = r[a];
        for (int b = 0; b < a; ++b) s -= L_omega[a * p + b] * v[b];
        v[a] = s / L_omega[a * p + a];
    }
    double d = 0.0;
    for (int a = 0; a < p; ++a) d += v[a] * v[a];
    const double logphi = -0.5 * p * log(2.0 * ORC_PI) - 0.5 * logdet - 0.5 * d;
    out[1] = 0.0;
    out[2] = 1.0;
    if (q == 0) { out[0] = logphi; return ORC_OK; }      /* Gaussian component */
    double c[QMAX];
    for (int k = 0; k < q; ++k) {
        double s = 0.0;
        for (int a = 0; a < p; ++a) s += A[k * p + a] * r[a];
        c[k] = s;
    }
    const double P = phi_r(q, c, Lambda, L, ones, min_key_gap);
    const int PW = 3 + q + q * q;
    if (!(P >= ORC_TMIN)) {                  /* reading A16 */
        out[0] = -INFINITY;
        for (int k = 3; k < PW; ++k) out[k] = 0.0;
        return ORC_OK;
    }
    const int q1 = q - 1;
    double phi[QMAX], Tk[QMAX], h[QMAX], ct[QMAX][QMAX], St[QMAX][QMAX * QMAX];
    int oth[QMAX][QMAX];
    for (int k = 0; k < q; ++k) {
        const double skk = Lambda[k * q + k];
        phi[k] = exp(norm_logpdf0(c[k], skk));
        Tk[k] = 1.0;
        if (q >= 2) {
            int na = 0;
            for (int t = 0; t < q; ++t) if (t != k) oth[k][na++] = t;
            for (int a = 0; a < q1; ++a) {
                const int ia = oth[k][a];
                ct[k][a] = c[ia] - Lambda[ia * q + k] * c[k] / skk;
                for (int b = 0; b < q1; ++b) {
                    const int ib = oth[k][b];
                    St[k][a * q1 + b] = Lambda[ia * q + ib] - Lambda[ia * q + k] * Lambda[k * q + ib] / skk;
                }
            }
            Tk[k] = phi_r(q1, ct[k], St[k], L, ones, min_key_gap);
        }
        h[k] = phi[k] * Tk[k];
    }
    double E1[QMAX];
    for (int a = 0; a < q; ++a) {
        double s = c[a] * P;
        for (int k = 0; k < q; ++k) s += Lambda[a * q + k] * h[k];
        E1[a] = s;
    }
    double G[QMAX * QMAX], BG[QMAX * QMAX];
    memset(G, 0, sizeof(G));
    memset(BG, 0, sizeof(BG));
    if (q >= 2) {
        const int q2 = q - 2;
        double Tkt[QMAX][QMAX];
        for (int k = 0; k < q; ++k)
            for (int t = k + 1; t < q; ++t) {
                double val = 1.0;
                if (q2 >= 1) {
                    int at = -1;
                    for (int a = 0; a < q1; ++a) if (oth[k][a] == t) at = a;
                    const double saa = St[k][at * q1 + at];
                    double ch[QMAX], Sh[QMAX * QMAX];
                    int rest[QMAX], nr = 0;
                    for (int a = 0; a < q1; ++a) if (a != at) rest[nr++] = a;
                    for (int a = 0; a < q2; ++a) {
                        const int ra = rest[a];
                        ch[a] = ct[k][ra] - St[k][ra * q1 + at] * ct[k][at] / saa;
                        for (int b = 0; b < q2; ++b) {
                            const int rb = rest[b];
                            Sh[a * q2 + b] = St[k][ra * q1 + rb] - St[k][ra * q1 + at] * St[k][at * q1 + rb] / saa;
                        }
                    }
                    val = phi_r(q2, ch, Sh, L, ones, min_key_gap);
                }
                Tkt[k][t] = Tkt[t][k] = val;
            }
        for (int k = 0; k < q; ++k) {
            double hk[QMAX];
            for (int a = 0; a < q1; ++a) hk[a] = exp(norm_logpdf0(ct[k][a], St[k][a * q1 + a])) * Tkt[k][oth[k][a]];
            for (int a = 0; a < q1; ++a) {
                double s = ct[k][a] * Tk[k];
                for (int b = 0; b < q1; ++b) s += St[k][a * q1 + b] * hk[b];
                G[k * q + oth[k][a]] = phi[k] * s;
                if (bound) {
                    double sb = fabs(ct[k][a] * Tk[k]);
                    for (int b = 0; b < q1; ++b) sb += fabs(St[k][a * q1 + b] * hk[b]);
                    BG[k * q + oth[k][a]] = fabs(phi[k]) * sb;
                }
            }
        }
    }
    double E2[QMAX * QMAX];
    for (int a = 0; a < q; ++a)
        for (int b = 0; b < q; ++b) {
            double s = 0.0;
            for (int k = 0; k < q; ++k) s += Lambda[a * q + k] * (G[k * q + b] + (k == b ? P : 0.0));
            E2[a * q + b] = s + c[a] * E1[b];
        }
    out[0] = q * log(2.0) + logphi + log(P);
    for (int a = 0; a < q; ++a) out[3 + a] = E1[a] / P;
    for (int a = 0; a < q; ++a)
        for (int b = 0; b < q; ++b) out[3 + q + a * q + b] = 0.5 * (E2[a * q + b] + E2[b * q + a]) / P;
    if (bound) moment_bounds(q, c, Lambda, h, P, P, BG, 1.0, bound);
    return ORC_OK;
}

/* =====================================================================================
 * E-step over all observations: Eq. (3)-(4), Alg. 2
 * with the sums S0..S7 (reading A4) accumulated in ascending j.
 * ===================================================================================== */
typedef struct {
    double L[PMAX * PMAX], A[QMAX * PMAX], Lam[QMAX * QMAX], logdet, kappa;
    double *chi0, *chi1, *chi2, *lv0;
} comp_derived;

int orc_estep(int64_t n, int p, int q, int g, const double *y,
              const double *pi, const double *mu, const double *sigma,
              const double *delta, const double *nu, const orc_lattice *L,
              int nthreads, int flags, double *pair_out, double *stats, double *loglik,
              double *min_key_gap) {
    return orc_estep_b(n, p, q, g, y, pi, mu, sigma, delta, nu, L, nthreads, flags, pair_out, stats, loglik,
                       min_key_gap, NULL);
}

/* orc_estep plus, per pair, the running error bounds of e3 / e4 (moment_bounds; [n][g][q + q*q],
 * analytic estimator only, 0 elsewhere) for the parity harness. */
int orc_estep_b(int64_t n, int p, int q, int g, const double *y,
                const double *pi, const double *mu, const double *sigma,
                const double *delta, const double *nu, const orc_lattice *L,
                int nthreads, int flags, double *pair_out, double *stats, double *loglik,
                double *min_key_gap, double *bound_out) {
    if (p < 1 || p > PMAX || q < 0 || q > 6 || g < 1 || n < 0) return ORC_EINVAL;
    const int sn = (flags & ORC_FAMILY_SN) != 0;
    const int direct = (flags & ORC_DIRECT) != 0 && q >= 1;
    const int use_e1 = ((flags & ORC_E1_EXACT) || direct) && q >= 1 && !sn;   /* q = 0: R1 is already exact */
    const int need_lattice = q >= 2 || use_e1 || direct;
    const int need_s = direct ? q + 1 : (q > 1 ? q : 1);
    if (need_lattice && (L == NULL || L->M < 1 || L->s < need_s)) return ORC_EINVAL;
    comp_derived *cd = (comp_derived *)calloc(g, sizeof(comp_derived));
    int rc = ORC_OK;
    for (int i = 0; i < g && rc == ORC_OK; ++i) {
        rc = orc_derive(p, q, sigma + (size_t)i * p * p, delta + (size_t)i * p * q, nu[i],
                        cd[i].L, cd[i].A, cd[i].Lam, &cd[i].logdet, &cd[i].kappa);
        if (rc == ORC_OK && need_lattice) {
            const double m0 = nu[i] + p;
            cd[i].chi0 = (double *)malloc(sizeof(double) * L->M);
            cd[i].chi1 = (double *)malloc(sizeof(double) * L->M);
            cd[i].chi2 = (double *)malloc(sizeof(double) * L->M);
            if (sn) {                                    /* normal SOV: every radius node = 1 */
                for (int64_t l = 0; l < L->M; ++l) cd[i].chi0[l] = cd[i].chi1[l] = cd[i].chi2[l] = 1.0;
            } else {
                orc_chi_table(L, m0, cd[i].chi0);
                orc_chi_table(L, m0 + 1.0, cd[i].chi1);
                orc_chi_table(L, m0 + 2.0, cd[i].chi2);
            }
            if (use_e1) {
                cd[i].lv0 = (double *)malloc(sizeof(double) * L->M);
                orc_logchi_table(L, m0, cd[i].lv0);
            }
        }
    }
    const int PW = 3 + q + q * q;        /* orc_pair output width */
    const int K = orc_k_stats(p, q);
    if (stats) memset(stats, 0, sizeof(double) * ((size_t)g * K + 1));
    double ll = 0.0;
    const int64_t CH = 4096;
    double *buf = (double *)malloc(sizeof(double) * (size_t)CH * g * PW);
    double *gaps = (double *)malloc(sizeof(double) * (size_t)CH * g);
    const int BW = q + q * q;            /* bound width per pair */
    double *bnd = bound_out ? (double *)calloc((size_t)CH * g * (BW > 0 ? BW : 1), sizeof(double)) : NULL;
    for (int64_t j0 = 0; j0 < n && rc == ORC_OK; j0 += CH) {
        const int64_t cnt = (n - j0 < CH) ? n - j0 : CH;
        int prc = ORC_OK;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
#endif
        for (int64_t jj = 0; jj < cnt * g; ++jj) {
            const int64_t j = j0 + jj / g;
            const int i = (int)(jj % g);
            double gap = INFINITY;
            const int r2 = direct ? orc_pair_direct(p, q, y + (size_t)j * p, mu + (size_t)i * p, cd[i].L, cd[i].A,
                                                    cd[i].Lam, nu[i], cd[i].kappa, cd[i].logdet, sn, L, cd[i].chi0,
                                                    cd[i].lv0, buf + (size_t)jj * PW, &gap)
                         : sn ? orc_pair_sn(p, q, y + (size_t)j * p, mu + (size_t)i * p, cd[i].L, cd[i].A,
                                            cd[i].Lam, cd[i].logdet, L, cd[i].chi0, buf + (size_t)jj * PW, &gap,
                                            bnd ? bnd + (size_t)jj * BW : NULL)
                              : orc_pair(p, q, y + (size_t)j * p, mu + (size_t)i * p, cd[i].L, cd[i].A,
                                         cd[i].Lam, nu[i], cd[i].kappa, L, cd[i].chi0, cd[i].chi1,
                                         cd[i].chi2, cd[i].lv0, buf + (size_t)jj * PW, &gap,
                                         bnd ? bnd + (size_t)jj * BW : NULL);
            gaps[jj] = gap;
            if (r2 != ORC_OK) prc = r2;
        }
        if (prc != ORC_OK) { rc = prc; break; }
        for (int64_t jj = 0; jj < cnt; ++jj) {        /* serial, ascending j */
            const int64_t j = j0 + jj;
            const double *yj = y + (size_t)j * p;
            double lf[16], mx = -INFINITY;
            for (int i = 0; i < g; ++i) {
                lf[i] = log(pi[i]) + buf[(size_t)(jj * g + i) * PW + 0];
                if (lf[i] > mx) mx = lf[i];
            }
            if (mx == -INFINITY) { rc = ORC_EUNDERFLOW; break; }
            double se = 0.0;
            for (int i = 0; i < g; ++i) se += exp(lf[i] - mx);
            const double lse = mx + log(se);
            ll += lse;
            for (int i = 0; i < g; ++i) {
                const double *o = buf + (size_t)(jj * g + i) * PW;
                const double tau = exp(lf[i] - lse);
                if (min_key_gap && gaps[jj * g + i] < min_key_gap[j * g + i]) min_key_gap[j * g + i] = gaps[jj * g + i];
                if (bnd)
                    for (int k = 0; k < BW; ++k) bound_out[((size_t)j * g + i) * BW + k] = bnd[(size_t)(jj * g + i) * BW + k];
                if (pair_out) {
                    double *po = pair_out + ((size_t)j * g + i) * (PW + 1);
                    po[0] = lf[i];
                    po[1] = tau;
                    for (int k = 1; k < PW; ++k) po[1 + k] = o[k];
                }
                if (!stats || !(tau > 0.0)) continue;
                double *S = stats + (size_t)i * K;
                const double e1me2 = o[1], e2 = o[2];
                const double *e3 = o + 3, *e4 = o + 3 + q;
                int off = 0;
                S[off++] += tau;                                       /* S0 */
                S[off++] += tau * e2;                                  /* S1 */
                for (int a = 0; a < p; ++a) S[off++] += tau * e2 * yj[a];               /* S2 */
                for (int a = 0; a < p; ++a)
                    for (int b = a; b < p; ++b) S[off++] += tau * e2 * yj[a] * yj[b];   /* S3 */
                for (int k = 0; k < q; ++k) S[off++] += tau * e3[k];                    /* S4 */
                for (int k = 0; k < q; ++k)
                    for (int l = k; l < q; ++l) S[off++] += tau * e4[k * q + l];        /* S5 */
                for (int a = 0; a < p; ++a)
                    for (int k = 0; k < q; ++k) S[off++] += tau * yj[a] * e3[k];        /* S6 */
                S[off++] += tau * e1me2;                               /* S7 */
            }
            if (rc != ORC_OK) break;
        }
    }
    if (stats) stats[(size_t)g * K] = ll;
    if (loglik) *loglik = ll;
    free(buf);
    free(gaps);
    free(bnd);
    for (int i = 0; i < g; ++i) { free(cd[i].chi0); free(cd[i].chi1); free(cd[i].chi2); free(cd[i].lv0); }
    free(cd);
    return rc;
}

/* =====================================================================================
 * M-step (Alg. 3), ECM order (reading A6):
 *   mu    <- (S2 - Delta_old S4) / S1
 *   B     <- S6 - mu S4'
 *   Delta <- B S5^{-1}
 *   Sigma <- [S3 - S2 mu' - mu S2' + S1 mu mu' - B Delta' - Delta B' + Delta S5 Delta'] / S0
 *   nu    <- root of log(nu/2) - psi(nu/2) + 1 + S7/S0 on [nu_lo, nu_hi] (reading A7)
 *   pi    <- S0 / n_total, floored at 1e-10, renormalised
 * ===================================================================================== */
static double nu_eq(double nu, double c) { return log(0.5 * nu) - orc_digamma(0.5 * nu) + 1.0 + c; }

int orc_mstep(int p, int q, int g, double n_total, const double *stats,
              double *pi, double *mu, double *sigma, double *delta, double *nu,
              double nu_lo, double nu_hi, int flags) {
    const int K = orc_k_stats(p, q);
    for (int i = 0; i < g; ++i) {
        const double *S = stats + (size_t)i * K;
        const double S0 = S[0], S1 = S[1];
        const double *S2 = S + 2, *S3p = S + 2 + p, *S4 = S3p + p * (p + 1) / 2;
        const double *S5p = S4 + q, *S6 = S5p + q * (q + 1) / 2;
        const double S7 = S6[p * q];
        if (!(S0 >= 1e-10)) return ORC_EEMPTY;
        double S3[PMAX * PMAX], S5[QMAX * QMAX];
        int off = 0;
        for (int a = 0; a < p; ++a)
            for (int b = a; b < p; ++b) { S3[a * p + b] = S3[b * p + a] = S3p[off++]; }
        off = 0;
        for (int k = 0; k < q; ++k)
            for (int l = k; l < q; ++l) { S5[k * q + l] = S5[l * q + k] = S5p[off++]; }
        double *mui = mu + (size_t)i * p, *Si = sigma + (size_t)i * p * p, *Di = delta + (size_t)i * p * q;
        for (int a = 0; a < p; ++a) {
            double s = S2[a];
            for (int k = 0; k < q; ++k) s -= Di[a * q + k] * S4[k];
            mui[a] = s / S1;
        }
        double B[PMAX * QMAX];
        for (int a = 0; a < p; ++a)
            for (int k = 0; k < q; ++k) B[a * q + k] = S6[a * q + k] - mui[a] * S4[k];
        if (q > 0) {
            double L5[QMAX * QMAX];
            if (chol(q, S5, L5) != ORC_OK) return ORC_ENOTPD;
            for (int a = 0; a < p; ++a) {
                double x[QMAX];
                for (int k = 0; k < q; ++k) x[k] = B[a * q + k];
                chol_solve(q, L5, x);                                  /* row a of B S5^{-1} */
                for (int k = 0; k < q; ++k) Di[a * q + k] = x[k];
            }
        }
        for (int a = 0; a < p; ++a)
            for (int b = 0; b < p; ++b) {
                double s = S3[a * p + b] - S2[a] * mui[b] - mui[a] * S2[b] + S1 * mui[a] * mui[b];
                for (int k = 0; k < q; ++k) s -= B[a * q + k] * Di[b * q + k] + Di[a * q + k] * B[b * q + k];
                for (int k = 0; k < q; ++k)
                    for (int l = 0; l < q; ++l) s += Di[a * q + k] * S5[k * q + l] * Di[b * q + l];
                Si[a * p + b] = s / S0;
            }
        for (int a = 0; a < p; ++a)
            for (int b = a + 1; b < p; ++b) {
                const double s = 0.5 * (Si[a * p + b] + Si[b * p + a]);
                Si[a * p + b] = Si[b * p + a] = s;
            }
        double Lt[PMAX * PMAX];
        if (chol(p, Si, Lt) != ORC_OK) {                              /* ridge repair */
            double md = 0.0;
            for (int a = 0; a < p; ++a) md += Si[a * p + a];
            md /= p;
            for (int a = 0; a < p; ++a) Si[a * p + a] += 1e-8 * md;
            if (chol(p, Si, Lt) != ORC_OK) return ORC_ENOTPD;
        }
        /* nu: log(nu/2) - psi(nu/2) decreases from +inf to 0; the skew-normal family has no nu */
        const double cst = S7 / S0;
        if (flags & ORC_FAMILY_SN) continue;
        if (nu_eq(nu_hi, cst) > 0.0) nu[i] = nu_hi;
        else if (nu_eq(nu_lo, cst) < 0.0) nu[i] = nu_lo;
        else {
            double lo = nu_lo, hi = nu_hi;
            for (int it = 0; it < 400; ++it) {
                const double mid = 0.5 * (lo + hi);
                if (nu_eq(mid, cst) > 0.0) lo = mid; else hi = mid;
                if (hi - lo <= 1e-12 * 0.5 * (lo + hi)) break;
            }
            nu[i] = 0.5 * (lo + hi);
        }
    }
    double tot = 0.0;
    for (int i = 0; i < g; ++i) {
        double pv = stats[(size_t)i * K] / n_total;
        if (pv < 1e-10) pv = 1e-10;
        pi[i] = pv;
        tot += pv;
    }
    for (int i = 0; i < g; ++i) pi[i] /= tot;
    return ORC_OK;
}

/* Alg. 4 with the typo readings of A8 and SPEC.md:338 guards. */
int orc_aitken_stop(double l_km2, double l_km1, double l_k, double tol) {
    const double den = l_km1 - l_km2;
    if (fabs(den) < 1e-300) return 1;
    const double a = (l_k - l_km1) / den;
    if (a >= 1.0) return 0;
    const double linf = l_km1 + (l_k - l_km1) / (1.0 - a);
    return fabs(linf - l_k) < tol;
}

/* O13: E-step at Psi^(0) gives l^(0); then [M-step, E-step] per iteration. */
int orc_fit(int64_t n, int p, int q, int g, const double *y, double *pi, double *mu,
            double *sigma, double *delta, double *nu, const orc_lattice *L,
            int nthreads, int flags, int max_iter, double tol, double nu_lo, double nu_hi,
            double *trace, int *n_iter, int *converged) {
    const int K = orc_k_stats(p, q);
    double *stats = (double *)malloc(sizeof(double) * ((size_t)g * K + 1));
    *n_iter = 0;
    *converged = 0;
    int rc = orc_estep(n, p, q, g, y, pi, mu, sigma, delta, nu, L, nthreads, flags, NULL, stats, &trace[0], NULL);
    for (int k = 1; k <= max_iter && rc == ORC_OK; ++k) {
        rc = orc_mstep(p, q, g, (double)n, stats, pi, mu, sigma, delta, nu, nu_lo, nu_hi, flags);
        if (rc != ORC_OK) break;
        rc = orc_estep(n, p, q, g, y, pi, mu, sigma, delta, nu, L, nthreads, flags, NULL, stats, &trace[k], NULL);
        if (rc != ORC_OK) break;
        *n_iter = k;
        if (tol > 0.0 && k >= 2 && orc_aitken_stop(trace[k - 2], trace[k - 1], trace[k], tol)) {
            *converged = 1;
            break;
        }
    }
    free(stats);
    return rc;
}

/* =====================================================================================
 * Alg. 1: parallel multi-start initialisation (NEXT-1).
 * The paper leaves open how the m partitions and Psi^(0) are made ("k-means or random
 * partitions", "computes Psi^(0) based on the given initial partition"); the readings I1-I4
 * of DESIGN.md §3 fix them:
 *   I1 random partitions: label_j = (splitmix64(splitmix64(splitmix64(seed) ^ stream) ^ j) >> 32)
 *      mod g, stream = l + m * attempt; redrawn (attempt + 1) while a component has < p+1 members.
 *   I2 k-means: first centre y_{j*}, j* = splitmix64(seed ^ 0xA5A5A5A5A5A5A5A5) mod n; centre k
 *      = argmax_j min_{c<k} |y_j - centre_c|^2 (farthest point, ties -> lowest j); Lloyd
 *      iterations (nearest centre, ties -> lowest index; centre = member mean; an empty cluster
 *      is re-seeded to the point farthest from its centre) until no label changes or `iters`.
 *      Squared distances are accumulated as d = fma(t, t, d) over ascending coordinates.
 *   I3 Psi^(0) from a partition: pi_i = n_i / n, ybar_i, S_i = (1/n_i) sum (y - ybar)(y - ybar)',
 *      gamma_ik = (1/n_i) sum (y_k - ybar_k)^3; Delta_i[k][k] = 0.5 sgn(gamma_ik) sqrt(S_ikk) for
 *      k < min(p, q) (0 elsewhere), mu_i = ybar_i - sqrt(2/pi) Delta_i 1_q, Sigma_i = S_i,
 *      nu_i = 10.  Invalid (candidate skipped) if n_i < p+1 or S_i is not PD.
 *   I4 selection: the LARGEST l^(0) (reading A9), ties -> lowest candidate index; with r > 0
 *      burn-in EM iterations the candidate's l is the log-likelihood after them.
 * ===================================================================================== */
uint64_t orc_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

int orc_random_label(uint64_t seed, int64_t stream, int64_t j, int g) {
    const uint64_t h = orc_splitmix64(orc_splitmix64(orc_splitmix64(seed) ^ (uint64_t)stream) ^ (uint64_t)j);
    return (int)((h >> 32) % (uint64_t)g);
}

int orc_random_partition(int64_t n, int p, int g, uint64_t seed, int l, int m, int32_t *labels) {
    int64_t cnt[16];
    for (int attempt = 0; attempt < 1000; ++attempt) {
        for (int i = 0; i < g; ++i) cnt[i] = 0;
        for (int64_t j = 0; j < n; ++j) {
            labels[j] = orc_random_label(seed, (int64_t)l + (int64_t)m * attempt, j, g);
            cnt[labels[j]]++;
        }
        int ok = 1;
        for (int i = 0; i < g; ++i) if (cnt[i] < p + 1) ok = 0;
        if (ok) return attempt;
    }
    return ORC_EINVAL;   /* PartitionInfeasible */
}

static double sqdist(int p, const double *a, const double *b) {
    double d = 0.0;
    for (int k = 0; k < p; ++k) {
        const double t = a[k] - b[k];
        d = fma(t, t, d);
    }
    return d;
}

int orc_kmeans(int64_t n, int p, int g, const double *y, uint64_t seed, int iters, int32_t *labels,
               double *centers) {
    if (n < g) return ORC_EINVAL;
    double *mind = (double *)malloc(sizeof(double) * n);
    const int64_t j0 = (int64_t)(orc_splitmix64(seed ^ 0xA5A5A5A5A5A5A5A5ULL) % (uint64_t)n);
    memcpy(centers, y + j0 * p, sizeof(double) * p);
    for (int64_t j = 0; j < n; ++j) mind[j] = sqdist(p, y + j * p, centers);
    for (int k = 1; k < g; ++k) {                       /* farthest point */
        int64_t best = 0;
        for (int64_t j = 1; j < n; ++j) if (mind[j] > mind[best]) best = j;
        memcpy(centers + k * p, y + best * p, sizeof(double) * p);
        for (int64_t j = 0; j < n; ++j) {
            const double d = sqdist(p, y + j * p, centers + k * p);
            if (d < mind[j]) mind[j] = d;
        }
    }
    for (int64_t j = 0; j < n; ++j) labels[j] = -1;
    for (int it = 0; it < iters; ++it) {
        int64_t changed = 0;
        for (int64_t j = 0; j < n; ++j) {                /* assignment */
            int bi = 0;
            double bd = sqdist(p, y + j * p, centers);
            for (int i = 1; i < g; ++i) {
                const double d = sqdist(p, y + j * p, centers + i * p);
                if (d < bd) { bd = d; bi = i; }
            }
            if (labels[j] != bi) { labels[j] = bi; ++changed; }
            mind[j] = bd;
        }
        if (changed == 0) break;
        double sum[16 * PMAX];
        int64_t cnt[16];
        memset(sum, 0, sizeof(sum));
        memset(cnt, 0, sizeof(cnt));
        for (int64_t j = 0; j < n; ++j) {                /* update */
            cnt[labels[j]]++;
            for (int k = 0; k < p; ++k) sum[labels[j] * p + k] += y[j * p + k];
        }
        for (int i = 0; i < g; ++i) {
            if (cnt[i] > 0) {
                for (int k = 0; k < p; ++k) centers[i * p + k] = sum[i * p + k] / (double)cnt[i];
            } else {                                      /* empty: re-seed to the farthest point */
                int64_t best = 0;
                for (int64_t j = 1; j < n; ++j) if (mind[j] > mind[best]) best = j;
                memcpy(centers + i * p, y + best * p, sizeof(double) * p);
                mind[best] = 0.0;
            }
        }
    }
    free(mind);
    return ORC_OK;
}

int orc_partition_params(int64_t n, int p, int q, int g, const double *y, const int32_t *labels,
                         double n_total, double *pi, double *mu, double *sigma, double *delta, double *nu) {
    for (int i = 0; i < g; ++i) {
        int64_t ni = 0;
        double ybar[PMAX] = {0};
        for (int64_t j = 0; j < n; ++j)
            if (labels[j] == i) {
                ++ni;
                for (int k = 0; k < p; ++k) ybar[k] += y[j * p + k];
            }
        if (ni < p + 1) return ORC_EINVAL;
        for (int k = 0; k < p; ++k) ybar[k] /= (double)ni;
        double S[PMAX * PMAX] = {0}, gam[PMAX] = {0};
        for (int64_t j = 0; j < n; ++j)
            if (labels[j] == i) {
                double t[PMAX];
                for (int k = 0; k < p; ++k) t[k] = y[j * p + k] - ybar[k];
                for (int a = 0; a < p; ++a) {
                    for (int b = 0; b < p; ++b) S[a * p + b] += t[a] * t[b];
                    gam[a] += t[a] * t[a] * t[a];
                }
            }
        for (int a = 0; a < p * p; ++a) S[a] /= (double)ni;
        double Lt[PMAX * PMAX];
        if (chol(p, S, Lt) != ORC_OK) return ORC_ENOTPD;
        double *Di = delta + (size_t)i * p * q;
        for (int a = 0; a < p * q; ++a) Di[a] = 0.0;
        for (int k = 0; k < p && k < q; ++k) Di[k * q + k] = (gam[k] < 0.0 ? -0.5 : 0.5) * sqrt(S[k * p + k]);
        for (int a = 0; a < p; ++a) {
            double s = 0.0;
            for (int k = 0; k < q; ++k) s += Di[a * q + k];
            mu[i * p + a] = ybar[a] - sqrt(2.0 / ORC_PI) * s;
        }
        memcpy(sigma + (size_t)i * p * p, S, sizeof(double) * p * p);
        nu[i] = 10.0;
        pi[i] = (double)ni / n_total;
    }
    return ORC_OK;
}

/* Alg. 1 lines 3-12 for given partitions: Psi^(0) (I3), optional r burn-in EM iterations,
 * l per candidate (-inf when invalid), selection I4.  params_out receive the winner's Psi. */
int orc_init_select(int64_t n, int p, int q, int g, const double *y, int m, const int32_t *labels,
                    const orc_lattice *L, int nthreads, int flags, int burn_in, double *loglik0, int *best,
                    double *pi, double *mu, double *sigma, double *delta, double *nu) {
    double *cp = (double *)malloc(sizeof(double) * (size_t)(g * (1 + p + p * p + p * (q > 0 ? q : 1) + 1)));
    double *bpi = cp, *bmu = bpi + g, *bsg = bmu + (size_t)g * p, *bde = bsg + (size_t)g * p * p;
    double *bnu = bde + (size_t)g * p * (q > 0 ? q : 1);
    *best = -1;
    for (int c = 0; c < m; ++c) {
        loglik0[c] = -INFINITY;
        int rc = orc_partition_params(n, p, q, g, y, labels + (size_t)c * n, (double)n, bpi, bmu, bsg, bde, bnu);
        if (rc != ORC_OK) continue;
        double ll;
        if (burn_in > 0) {
            double *trace = (double *)malloc(sizeof(double) * (burn_in + 1));
            int ni = 0, cv = 0;
            rc = orc_fit(n, p, q, g, y, bpi, bmu, bsg, bde, bnu, L, nthreads, flags, burn_in, 0.0, 0.1, 1000.0,
                         trace, &ni, &cv);
            ll = trace[ni];
            free(trace);
        } else {
            rc = orc_estep(n, p, q, g, y, bpi, bmu, bsg, bde, bnu, L, nthreads, flags, NULL, NULL, &ll, NULL);
        }
        if (rc != ORC_OK || !(ll > -INFINITY)) continue;
        loglik0[c] = ll;
        if (*best < 0 || ll > loglik0[*best]) {
            *best = c;
            memcpy(pi, bpi, sizeof(double) * g);
            memcpy(mu, bmu, sizeof(double) * g * p);
            memcpy(sigma, bsg, sizeof(double) * g * p * p);
            if (q > 0) memcpy(delta, bde, sizeof(double) * g * p * q);
            memcpy(nu, bnu, sizeof(double) * g);
        }
    }
    free(cp);
    return *best >= 0 ? ORC_OK : ORC_EINVAL;
}
