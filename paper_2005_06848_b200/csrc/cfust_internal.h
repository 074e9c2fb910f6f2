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
    double *stats;                  // [g*K+1] reduced (then all-reduced) statistics
    int *status;                    // [4]: 0 E-step underflow, 1 M-step/derive error code
    double nu_lo, nu_hi;
    int M;                          // lattice points (0 when q <= 1)
    uint32_t z[8];
    double shift[8];
    int num_sms;
    int e1_exact;                   // 1: exact e1 = E[log W | y] (reading R2'); 0: reading A5
};

// rows of the per-component node table DevState::chi
constexpr int CHI_M1 = 1, CHI_M2 = 2, CHI_LV = 3, CHI_ROWS = 4;

// Launchers (all asynchronous on `st`); return cudaError_t as int.
int launch_estep(const DevState &s, int mode, const int64_t *idx, int64_t cnt, double *pair_out,
                 cudaStream_t st, int *nblocks_out);
int launch_reduce(const DevState &s, int nblocks, int mode, double *out, cudaStream_t st);
int launch_mstep(const DevState &s, cudaStream_t st);
int launch_derive(const DevState &s, cudaStream_t st);
int launch_chi(const DevState &s, cudaStream_t st);
int launch_lattice(const DevState &s, cudaStream_t st);
int launch_check_finite(const double *y, int64_t count, int *flag, cudaStream_t st);
size_t comp_dev_size();
int upload_special_constants();
int launch_special(int which, const double *x, double *y, int64_t n, double aux, cudaStream_t st);
int max_partial_blocks(const DevState &s);

}  // namespace cfust
