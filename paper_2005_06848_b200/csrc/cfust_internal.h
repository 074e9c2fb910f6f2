// cfust_internal.h — host-side interface between the C ABI (cfust_abi.cu) and the kernels
// (cfust_kernels.cu).  Not part of the public ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cfust {

struct LatticeDev;
struct CompDev;

// Device-resident state of one rank (all pointers are device memory owned by the context,
// except y when the caller attached its own device buffer).
struct DevState {
    int p, q, g, K;                 // K = sufficient statistics per component
    int64_t n;                      // local observations
    double n_total;                 // global n (pi update)
    const double *y;                // [n][p]
    double *pi, *mu, *sigma, *delta, *nu;   // Psi on device
    CompDev *comp;                  // [g]
    double *chi;                    // [g][CHI_ROWS][M]: chi radius nodes for df m0, m0+1, m0+2; log V (df m0)
    double *W;                      // [q][M] lattice coordinates (fixed per context)
    double *partials;               // [max_blocks][g*K+1]
    double *stats;                  // [g*K+2] reduced (then all-reduced): statistics, l, underflow flag
    int *status;                    // [4]: 0 E-step underflow, 1 M-step/derive error code, 2 non-finite y
    double *trace;                  // [TRACE_CAP] l^(k) recorded by the M-step during cfust_fit (or NULL)
    int *fitctl;                    // [3] fit bookkeeping (mstep_fused_kernel), NULL outside cfust_fit
    double nu_lo, nu_hi;
    int M;                          // lattice points (0 when q <= 1)
    uint32_t z[8];
    double shift[8];
    int num_sms;
    int e1_exact;                   // 1: exact e1 = E[log W | y] (reading R2'); 0: reading A5
    int family;                     // 0: skew-t (CFUST); 1: skew-normal (CFUSN, nu = inf; q = 0: Gaussian)
    int direct;                     // 1: SOV-direct truncated moments (reading D1); 0: analytic (O6-O7)
    int nw;                         // lattice coordinates tabulated in W (rows)
    int split_force;                // warps per observation for small n: 0 auto, 1/2/4/8 forced (env CFUST_SPLIT)
    double *tau_out;                // density pass (mode 1): responsibilities [n][g] if non-NULL
    int32_t *label_out;             // density pass (mode 1): argmax_i tau_ij [n] if non-NULL
    int *wperm;                     // [M] lattice points in ascending order of coordinate 0 (chi nodes)
};

constexpr int TRACE_CAP = 4096;   // device trace ring (power of two); cfust_fit drains it when full

// rows of the per-component node table DevState::chi
constexpr int CHI_M1 = 1, CHI_M2 = 2, CHI_LV = 3, CHI_ROWS = 4;

// Launchers (all asynchronous on `st`); return cudaError_t as int.
int launch_estep(const DevState &s, int mode, const int64_t *idx, int64_t cnt, double *pair_out,
                 cudaStream_t st, int *nblocks_out);
int launch_reduce(const DevState &s, int nblocks, int mode, double *out, cudaStream_t st);
int mstep_launches();
int launch_mstep(const DevState &s, cudaStream_t st);
int launch_derive(const DevState &s, cudaStream_t st);
int launch_chi(const DevState &s, cudaStream_t st);
int launch_lattice(const DevState &s, cudaStream_t st);
int launch_check_finite(const double *y, int64_t count, int *flag, cudaStream_t st);
size_t comp_dev_size();
int upload_special_constants();
int launch_special(int which, const double *x, double *y, int64_t n, double aux, cudaStream_t st);
int max_partial_blocks(const DevState &s);

// Alg. 1 (cfust_init.cu)
int launch_random_labels(int32_t *lab, int64_t n, int64_t j0, int g, uint64_t seed, int64_t stream, cudaStream_t st);
int launch_mind(const double *y, int64_t n, int p, const double *c, double *mind, int init, cudaStream_t st);
int launch_argmax(const double *v, int64_t n, int64_t j0, double *scratch, double *out, cudaStream_t st);
int launch_assign(const double *y, int64_t n, int p, int g, const double *cen, int32_t *lab, double *mind,
                  double *partials, int *nb_out, cudaStream_t st);
int part_sums_width(int p, int g, int pass);
int launch_part_sums(const double *y, int64_t n, int p, int g, const int32_t *lab, const double *ybar, int pass,
                     int max_blocks, double *partials, int *nb_out, cudaStream_t st);
int launch_centers(const double *sums1, int p, int g, double *out, int *empty, cudaStream_t st);
int launch_partition_params(const DevState &s, const double *sums1, const double *sums2, const double *ybar, int *valid,
                            cudaStream_t st);
int launch_reduce_cols(const double *partials, int nblocks, int stride, int ncols, double *out, cudaStream_t st);

}  // namespace cfust
