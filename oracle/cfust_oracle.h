/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, double-precision CPU implementation of the FM-CFUST EM iteration
 * (Lee, McLachlan & Leemaqz, arXiv 2005.06848).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_2005_06848_b200/csrc);
 * both receive the data, parameters and lattice inputs (z, shift) from synth/.
 *
 * Every formula cites the passage it follows: PAPER.md line numbers, or the DESIGN.md
 * readings R-xx where the paper omits the E-/M-step.
 *
 * Parity-pin status (tests/test_oracle_*.py): every function below is pinned against
 * closed forms, scipy/mpmath library routines, quadrature, Monte Carlo or invariants;
 * see DESIGN.md §"Oracle pins".  No function is "parity unpinned".
 */
#ifndef CFUST_ORACLE_H
#define CFUST_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = -1, ORC_ENOTPD = -4, ORC_EUNDERFLOW = -5, ORC_EEMPTY = -6 };
/* E-step / fit flags: exact e1 (reading R2'); skew-normal family (CFUSN, nu = inf; reading F1) */
enum { ORC_E1_EXACT = 1, ORC_FAMILY_SN = 2, ORC_DIRECT = 4 };   /* ORC_DIRECT: SOV-direct moments (D1) */

typedef struct {
    int32_t M;            /* number of lattice points (power of two) */
    int32_t s;            /* number of coordinates available */
    const uint32_t *z;    /* generating vector [s] */
    const double *shift;  /* shift [s], in (0,1) */
} orc_lattice;

/* ---- special functions (pins: C12) ---- */
double orc_norm_cdf(double x);
double orc_norm_quantile(double u);
double orc_gamma_p(double a, double x);
double orc_gamma_q(double a, double x);
double orc_chi2_quantile(double w, double m);
double orc_ibeta(double a, double b, double x, double xc);
double orc_t_cdf(double x, double m);
double orc_t1_logpdf(double x, double loc, double s2, double m);
double orc_digamma(double x);

/* ---- lattice (O0) ---- */
double orc_lattice_w(const orc_lattice *L, int64_t l, int k);
void orc_chi_table(const orc_lattice *L, double m, double *s_out);
void orc_logchi_table(const orc_lattice *L, double m, double *out);   /* log chi2_m^{-1}(w_{l,0}) */

/* ---- T_r(b; 0, S, m) (O4, chi-normal SOV reading R-T) ---- */
double orc_Tr(int r, const double *b, const double *S, double m,
              const orc_lattice *L, const double *chi_s, double *min_key_gap);
/* the same lattice rule, also returning *wsum = (1/M) sum_l f_l lv_l (r = 1 on the lattice) */
double orc_Tr_w(int r, const double *b, const double *S, double m, const orc_lattice *L,
                const double *chi_s, const double *lv, double *min_key_gap, double *wsum);

/* ---- per-component derived quantities (O1) ---- */
int orc_derive(int p, int q, const double *sigma, const double *delta, double nu,
               double *L_omega, double *A, double *Lambda, double *logdet, double *kappa);

/* ---- per pair E-step quantities (O2-O8). out = [logf_noprior, e1me2, e2, e3(q), e4(q*q)]
 * lv_m0 (may be NULL): log chi2_{m0}^{-1} node table -> exact e1 = E[log W | y] (reading R2') ---- */
int orc_pair(int p, int q, const double *y, const double *mu, const double *L_omega,
             const double *A, const double *Lambda, double nu, double kappa,
             const orc_lattice *L, const double *chi_m0, const double *chi_m1,
             const double *chi_m2, const double *lv_m0, double *out, double *min_key_gap, double *bound);

/* ---- skew-normal pair (CFUSN, reading F1): ones = radius table of 1.0 (normal SOV) ---- */
int orc_pair_sn(int p, int q, const double *y, const double *mu, const double *L_omega,
                const double *A, const double *Lambda, double logdet, const orc_lattice *L,
                const double *ones, double *out, double *min_key_gap, double *bound);

/* ---- SOV-direct truncated-moment estimator (reading D1); sn: skew-normal family ---- */
int orc_pair_direct(int p, int q, const double *y, const double *mu, const double *L_omega,
                    const double *A, const double *Lambda, double nu, double kappa, double logdet, int sn,
                    const orc_lattice *L, const double *chi_m0, const double *lv_m0, double *out,
                    double *min_key_gap);

/* ---- E-step over n observations (O9-O10); flags: ORC_E1_EXACT, ORC_FAMILY_SN, ORC_DIRECT ----
 * pair_out (may be NULL): [n][g][4+q+q*q] = logf, tau, e1me2, e2, e3(q), e4(q*q)
 * stats (may be NULL): [g*K + 1], K = 3+p+p(p+1)/2+q+q(q+1)/2+p*q, last entry = loglik */
int orc_estep(int64_t n, int p, int q, int g, const double *y,
              const double *pi, const double *mu, const double *sigma,
              const double *delta, const double *nu, const orc_lattice *L,
              int nthreads, int flags, double *pair_out, double *stats, double *loglik,
              double *min_key_gap);
/* the same, plus bound_out (may be NULL): [n][g][q+q*q] running error bounds of e3 / e4 (parity
 * harness, reading P1; analytic estimator only) */
int orc_estep_b(int64_t n, int p, int q, int g, const double *y,
                const double *pi, const double *mu, const double *sigma,
                const double *delta, const double *nu, const orc_lattice *L,
                int nthreads, int flags, double *pair_out, double *stats, double *loglik,
                double *min_key_gap, double *bound_out);
/* reading A14 harness: 1 = sort near-tied reordering keys (within 1e-12 relative) in the opposite order */
void orc_set_tie_flip(int on);

/* ---- M-step (O11-O12), in place on the parameter arrays ---- */
int orc_mstep(int p, int q, int g, double n_total, const double *stats,
              double *pi, double *mu, double *sigma, double *delta, double *nu,
              double nu_lo, double nu_hi, int flags);

/* ---- Aitken stopping rule (Alg. 4; reading A8) ---- */
int orc_aitken_stop(double l_km2, double l_km1, double l_k, double tol);

/* ---- fit loop (O13): trace gets loglik^(0..n_iter) ---- */
int orc_fit(int64_t n, int p, int q, int g, const double *y, double *pi, double *mu,
            double *sigma, double *delta, double *nu, const orc_lattice *L,
            int nthreads, int flags, int max_iter, double tol, double nu_lo, double nu_hi,
            double *trace, int *n_iter, int *converged);

int orc_k_stats(int p, int q);

/* ---- Alg. 1, readings I1-I4 ---- */
uint64_t orc_splitmix64(uint64_t x);
int orc_random_label(uint64_t seed, int64_t stream, int64_t j, int g);
/* returns the attempt used (>= 0) or ORC_EINVAL when every attempt leaves a component < p+1 */
int orc_random_partition(int64_t n, int p, int g, uint64_t seed, int l, int m, int32_t *labels);
int orc_kmeans(int64_t n, int p, int g, const double *y, uint64_t seed, int iters, int32_t *labels,
               double *centers);
int orc_partition_params(int64_t n, int p, int q, int g, const double *y, const int32_t *labels,
                         double n_total, double *pi, double *mu, double *sigma, double *delta, double *nu);
int orc_init_select(int64_t n, int p, int q, int g, const double *y, int m, const int32_t *labels,
                    const orc_lattice *L, int nthreads, int flags, int burn_in, double *loglik0, int *best,
                    double *pi, double *mu, double *sigma, double *delta, double *nu);

#ifdef __cplusplus
}
#endif
#endif
