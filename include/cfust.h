/*
 * cfust.h — C ABI of the B200-native FM-CFUST EM hot path (libcfust.so).
 *
 * Implements the EM iteration for a g-component mixture of canonical fundamental skew-t
 * (CFUST) distributions, Eq. (2) of Lee, McLachlan & Leemaqz, arXiv 2005.06848
 * (PAPER.md:154-166), following the EM outline of PAPER.md:197-226 and the data-parallel
 * E-step / M-step split of Algorithms 2-3.  The E-/M-step formulas the
 * paper omits follow DESIGN.md §3 (readings R-E, R-M, R-T).
 *
 * Conventions
 *  - Every call returns int: CFUST_OK (0) or a negative CFUST_E* code; the message is
 *    available from cfust_last_error(ctx).  Not converging is not an error.
 *  - All arrays are FP64, row-major, C-contiguous.
 *  - Host pointers are only read during the call (copied); caller keeps ownership.
 *    Exception: with opts.y_on_device = 1, y is a DEVICE pointer that the caller owns and
 *    must keep alive and unchanged until cfust_destroy (it is not copied).
 *  - The context owns all device memory, its CUDA stream, events and (world > 1) the NCCL
 *    communicator until cfust_destroy.  No global state; one context per thread at a time.
 *  - Limits: 1 <= p <= 8, 0 <= q <= 6, 1 <= g <= 8; lattice M a power of two in
 *    [1024, 65536] when q >= 2 or (q == 1 and opts.e1_exact) or opts.estimator == 1; otherwise
 *    no lattice is used.  lattice_z / lattice_shift hold max(q, 1) entries (q + 1 with
 *    opts.estimator == 1).
 *  - There is no CPU fallback: without a CUDA device every call fails with CFUST_ECUDA.
 *  - Environment (optional): CFUST_SPLIT = 1|2|4|8 forces the warps per observation of the
 *    small-n E-step (read at cfust_em_init; default: chosen from n and the q-tuned occupancy);
 *    CFUST_NCCL_TIMEOUT_S = seconds bounds every collective wait (see CFUST_ENCCL).
 *  - Each call and E-/M-step phase is an NVTX range ("cfust_fit", "cfust:estep-kernel", ...).
 */
#ifndef CFUST_H
#define CFUST_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CFUST_OK 0
#define CFUST_EINVAL -1      /* bad argument (NULL, out of range, unsupported M)          */
#define CFUST_EDIM -2        /* DimensionMismatch (p, q, g, n inconsistent)     */
#define CFUST_EMIXPROP -3    /* pi_i <= 0 or |sum pi - 1| > 1e-12               */
#define CFUST_ENOTPD -4      /* Cholesky pivot <= 1e-300 in Sigma, Omega or S5 */
#define CFUST_EUNDERFLOW -5  /* all g component densities are 0 at some y_j   */
#define CFUST_EEMPTY -6      /* S0_i < 1e-10: empty component in the M-step    */
#define CFUST_ECUDA -7       /* CUDA runtime error / no device                               */
#define CFUST_ENCCL -8       /* NCCL error: a failed collective, an NCCL asynchronous error seen
                                while waiting (ncclCommGetAsyncError is polled), or a wait longer
                                than CFUST_NCCL_TIMEOUT_S seconds (environment; default 1800 s when
                                world > 1, unbounded for one rank).  The communicator is then
                                aborted and every later call on the context returns CFUST_ENCCL
                                (fail fast; no elastic recovery).  A local CUDA failure on a
                                multi-rank context also aborts the communicator, so the peers'
                                next collective fails instead of blocking.                      */

typedef struct cfust_ctx cfust_ctx;   /* opaque */

/* Mixture parameters Psi = (pi, mu, Sigma, Delta, nu).
 * Host buffers, caller-owned: pi[g], mu[g][p], sigma[g][p][p] (symmetric PD),
 * delta[g][p][q] (ignored / may be NULL when q == 0), nu[g] (> 0). */
typedef struct {
    double *pi;
    double *mu;
    double *sigma;
    double *delta;
    double *nu;
} cfust_params;

/* Options.  Zero-initialise and set what you need. */
typedef struct {
    int32_t lattice_m;             /* M: lattice points for T_r, r >= 2 (power of two)           */
    const uint32_t *lattice_z;     /* [q] rank-1 generating vector (host), reading A12            */
    const double *lattice_shift;   /* [q] seed-defined shift in (0,1) (host), reading A11          */
    double nu_lo, nu_hi;           /* nu bracket; 0,0 -> [0.1, 1000] (reading A7)                 */
    int32_t y_on_device;           /* 1: y is a caller-owned device pointer (not copied)          */
    int32_t device;                /* CUDA device ordinal; < 0 -> current device                  */
    int32_t rank, world;           /* world <= 1: single GPU (no NCCL unless nccl_id is given)     */
    const void *nccl_id;           /* 128-byte ncclUniqueId, identical on all ranks; required when
                                      world > 1; with world = 1 it creates a one-rank communicator
                                      so every collective path runs (tests)                       */
    int64_t n_total;               /* sum of n over ranks (pi = S0 / n_total); 0 -> n              */
    int32_t timing;                /* 1: record CUDA events per phase (see cfust_get_timing)       */
    int32_t e1_exact;              /* 0: e1 = E[log W|y] by the closed-form approximation (reading
                                      A5); 1: exact, estimated on T0's own lattice
                                      points as (sum_l f_l log V_l)/(sum_l f_l) - log rho (reading
                                      R2', NEXT-2).  With q = 1 this needs a lattice (lattice_m,
                                      lattice_z[1], lattice_shift[1]); with q = 0 it is a no-op.  */
    int64_t global_offset;         /* global index of this shard's first observation (j0; 0 for one
                                      rank): keys the random partitions and k-means seeding of Alg. 1 */
    int32_t family;                /* 0: skew-t components (CFUST, Eq. (2)); 1: skew-normal (CFUSN, the
                                      nu -> inf limit; reading F1): e2 = 1, nu is
                                      neither used nor updated; with q = 0 a Gaussian mixture
                                      (PAPER.md:147-151).  NEXT-3. */
    int32_t estimator;             /* truncated moments e3, e4: 0 = analytic reduction to T_{q-1},
                                      T_{q-2} integrals (DESIGN.md §3 R-E, default); 1 = SOV-direct
                                      (reading D1, NEXT-3): estimated on T0's own lattice points with
                                      the last coordinate drawn — 2q Phi/Phi^-1 per point instead of
                                      2(2q-1)+q(2q-3)+C(q,2)(2q-5); e1 is then exact.  Needs a lattice
                                      with q+1 coordinates (lattice_z/shift[q+1]) for every q >= 1.
                                      The density and tau are identical to estimator 0.  */
} cfust_opts;

typedef struct {
    int32_t n_iter;        /* EM iterations (M-steps) performed                              */
    int32_t converged;     /* 1 if the Aitken rule (Alg. 4) stopped the fit  */
    double *loglik_trace;  /* caller buffer [trace_cap]: l^(0..n_iter), l^(k) at Psi^(k)      */
    int32_t trace_cap;
    double wall_time_s;
} cfust_result;

/* Create a context on this rank's shard y[n][p] (observations j0..j0+n-1 of the global data;
 * contiguous blocks), upload Psi^(0) and derive Omega, Lambda, ...
 * Validates: y finite, pi (EMIXPROP), Sigma/Omega PD (ENOTPD), nu > 0. */
int cfust_em_init(cfust_ctx **out, const double *y, int64_t n, int32_t p, int32_t g, int32_t q,
                  const cfust_params *init, const cfust_opts *opts);

/* Replace the data shard (same n, p).  on_device = 0: host array, copied (H2D on the
 * context stream); 1: caller-owned device pointer, used in place. */
int cfust_set_data(cfust_ctx *ctx, const double *y, int32_t on_device);

/* E-step at the current Psi^(k) (Eq. (3)-(4), Alg. 2): tau, e1-e2, e2, e3, e4 per pair and the
 * eight sufficient statistics S0..S7 per component (reading A4), reduced over the shard and
 * (world > 1) all-reduced over ranks.  loglik_out (may be NULL) receives l^(k) = sum_j log f_j;
 * stats_out (may be NULL) receives the global vector [g*K + 1], K = cfust_k_stats(p, q):
 * per component [S0, S1, S2(p), S3(p(p+1)/2, upper row-major), S4(q), S5(q(q+1)/2),
 * S6(p*q row-major), S7], then l.  Blocks until the results are on the host if either is non-NULL. */
int cfust_estep(cfust_ctx *ctx, double *loglik_out, double *stats_out);

/* M-step (Alg. 3; reading R-M, ECM order) from the last E-step's statistics, entirely on the
 * device: mu, Delta, Sigma, nu (root of the nu equation by safeguarded Newton, reading A7), pi;
 * then re-derives Omega, Lambda, chi nodes.  Transactional: if any component fails (ENOTPD,
 * EEMPTY) no parameter of any component changes; it also refuses (parameters unchanged,
 * CFUST_EUNDERFLOW) when the E-step flagged an underflow on any rank. */
int cfust_mstep(cfust_ctx *ctx);

/* One EM iteration = cfust_estep + cfust_mstep; *loglik_out = l at the pre-M-step Psi.  Runs as
 * one CUDA graph (E-step kernel, reduction, the single all-reduce, M-step, chi nodes; captured on
 * first use, not with opts.timing) with one host synchronisation. */
int cfust_iterate(cfust_ctx *ctx, double *loglik_out);

/* Density-only pass (T0 only): l = sum_j log f(y_j; Psi) at the current Psi (Eq. (3)). */
int cfust_loglik(cfust_ctx *ctx, double *out);

/* Clustering output at the current Psi (density pass, as cfust_loglik): labels_out[n] (may be NULL)
 * receives the MAP component argmax_i tau_ij (ties -> lowest i; the hard partition of SPEC.md:72),
 * tau_out[n][g] (may be NULL) the responsibilities tau_ij of Eq. (4), loglik_out
 * (may be NULL) l.  Local observations of this rank; host buffers, caller-owned.  CFUST_EUNDERFLOW
 * as cfust_estep. */
int cfust_predict(cfust_ctx *ctx, int32_t *labels_out, double *tau_out, double *loglik_out);

/* Full fit: E-step, then max_iter x [M-step, E-step] with the Aitken stop when tol > 0
 * (Alg. 4, reading A8); out->loglik_trace gets l^(0..n_iter).  Each [M-step, E-step] is one CUDA
 * graph; the M-step records l on the device, so with tol <= 0 the whole fit runs with one host
 * synchronisation at the end, and with tol > 0 with one per iteration (l^(k) for the rule).  When
 * the fit runs to max_iter the last l comes from the density-only pass (cfust_loglik: same value,
 * no statistics), so call cfust_estep before a further cfust_mstep.  On an error the parameters are
 * those of the last successful M-step and out->n_iter / the trace follow that point (an E-step
 * underflow at Psi^(j): n_iter = j - 1; an M-step failure producing Psi^(j+1): n_iter = j). */
int cfust_fit(cfust_ctx *ctx, int32_t max_iter, double tol, cfust_result *out);

int cfust_get_params(cfust_ctx *ctx, cfust_params *out);         /* copies into caller buffers */
int cfust_set_params(cfust_ctx *ctx, const cfust_params *in);    /* validates, re-derives      */

/* ---- Alg. 1: parallel multi-start initialisation (NEXT-1; readings I1-I4 of
 * DESIGN.md §3) ----
 * cfust_init_partitions: step 1, the m candidate hard partitions of this rank's shard, made on the
 * device into a context-owned buffer [m][n] (int32 labels in [0, g)):
 *   candidate 0      k-means (reading I2): first centre y_{j*}, j* = splitmix64(seed ^
 *                    0xA5A5A5A5A5A5A5A5) mod n_total; farthest-point seeding; Lloyd iterations
 *                    (at most kmeans_iters) with empty clusters re-seeded to the farthest point;
 *   candidates 1..m-1  random labels (reading I1) splitmix64(splitmix64(splitmix64(seed) ^
 *                    (l + m a)) ^ j) >> 32 mod g for global index j, redrawn (a = 1, 2, ...)
 *                    while a component has fewer than p+1 members over all ranks.
 * labels_out (may be NULL): host [m][n] copy.  Errors: CFUST_EINVAL (m < 1, n_total < g, or no
 * feasible random partition within 1000 draws), CFUST_ECUDA, CFUST_ENCCL.  Collective over ranks.
 *
 * cfust_init_select: steps 2-12 for the m partitions (labels: host [m][n], or NULL for the buffer
 * of cfust_init_partitions).  Per candidate: Psi^(0) from the partition moments (reading I3) on the
 * device, `burn_in` EM iterations, then l = sum_j log f(y_j) (the density pass of cfust_loglik);
 * invalid candidates (a component with < p+1 members or a non-PD covariance) get -inf.  Selects
 * the LARGEST l (reading A9; ties -> lowest index), installs its Psi in the context and returns
 * loglik0_out[m] (may be NULL) and *best_out.  CFUST_EINVAL if every candidate is invalid. */
int cfust_init_partitions(cfust_ctx *ctx, int32_t m, uint64_t seed, int32_t kmeans_iters, int32_t *labels_out);
int cfust_init_select(cfust_ctx *ctx, int32_t m, const int32_t *labels, int32_t burn_in, double *loglik0_out,
                      int32_t *best_out);

/* Per-pair E-step outputs for observations idx[0..cnt) (local indices) at the current Psi,
 * for parity checks: out[cnt][g][4 + q + q*q] = log(pi_i f_ij), tau_ij, e1-e2, e2, e3(q), e4(q*q).
 * Does not touch the accumulated statistics. */
int cfust_get_pairs(cfust_ctx *ctx, const int64_t *idx, int64_t cnt, double *out);

/* Accumulated device time per phase since the last reset (opts.timing = 1):
 * ms[0] E-step kernel, ms[1] reduce, ms[2] all-reduce, ms[3] M-step+derive+chi nodes;
 * counts[0..3] launches per phase.  reset != 0 clears after reading. */
int cfust_get_timing(cfust_ctx *ctx, double *ms, int64_t *counts, int32_t reset);

/* The cudaStream_t the context launches on (as void*), for event timing by the caller. */
void *cfust_stream(cfust_ctx *ctx);

/* Kernel launches issued since creation (for bench's gpu_launches). */
int64_t cfust_launch_count(cfust_ctx *ctx);

/* Fill out[128] with a fresh ncclUniqueId (rank 0), to be broadcast to all ranks and passed
 * as opts.nccl_id.  Per EM iteration the ranks exchange exactly one NCCL all-reduce (sum, FP64) of
 * the vector [statistics (g*K), l, underflow flag]. */
int cfust_nccl_unique_id(void *out);

/* Diagnostic: evaluate a device special function element-wise on host arrays x[n] -> y[n]
 * (the exact code the kernels inline).  which: 0 Phi, 1 Phi^{-1}, 2 exp (x <= 0), 3 log
 * (0 < x <= 1), 4 univariate t CDF with df = aux, 5 chi-square quantile with df = aux,
 * 6 digamma, 7 sqrt, 8 trigamma (the M-step's nu Newton step), 9 log Gamma (x > 0, the M-step's
 * derived constants), 10 Phi and 11 Phi^{-1} with exp through the 2^(j/64) table (the SOV
 * loop's optional variant, CFUST_SOV_XT), 12 that table exp (x <= 709).  No context needed; CFUST_ECUDA
 * without a device. */
int cfust_eval_special(int32_t which, const double *x, double *y, int64_t n, double aux);

int cfust_k_stats(int32_t p, int32_t q);
const char *cfust_last_error(const cfust_ctx *ctx);
void cfust_destroy(cfust_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* CFUST_H */
