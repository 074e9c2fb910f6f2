// cfust_kernels.cu — FP64 CUDA kernels of the FM-CFUST EM hot path for sm_100a.
//
//   estep_cfust_kernel<Q,MODE,DIRECT>  q >= 1: one warp per observation j, looping over the g
//                               components; the M lattice points of every T_r are split
//                               over the 32 lanes and combined by xor-shuffle reductions
//                               (Alg. 2; formulas DESIGN.md §3).  MODE 0
//                               statistics, 1 density pass (log-likelihood, tau / MAP labels),
//                               2 per-pair dump; DIRECT = SOV-direct moments (reading D1).
//   estep_t_mma_kernel<G>       q == 0 (Delta = 0): warp per 32 observations,
//                               S3 by FP64 tensor-core MMA (default); estep_t_kernel<P> is the
//                               shared-memory register-blocked variant (CFUST_T_MMA=0).
//   reduce_kernel               deterministic column sums of the per-block partials.
//   mstep_kernel, mstep_derive_kernel  one warp per component: M-step (Alg. 3, PAPER.md:370-381;
//                               reading R-M), then pi and the derived quantities.
//   derive_kernel               Omega, chol, A, Lambda, constants.
//   chi_kernel                  chi radius nodes of the lattice for df m0, m0+1, m0+2 (+ log V).
//   lattice_kernel, check_finite_kernel, special_kernel (diagnostic), dump_t_kernel (q = 0 dump).
// Alg. 1 (multi-start initialisation) kernels live in cfust_init.cu.
//
// Tensor cores: only the q = 0 Gram contraction is a dense product (DMMA); everything else is
// scalar FP64 special-function integration (BASELINE.json north_star).
#include "cfust_device.cuh"
#include "cfust_internal.h"

#include <cstdio>

namespace cfust {

#ifndef CFUST_EW
#define CFUST_EW 8
#endif
#ifndef CFUST_MINB
#define CFUST_MINB 2
#endif
constexpr int EW = CFUST_EW;     // warps per block of the CFUST E-step
constexpr int MINB = CFUST_MINB; // resident blocks per SM the register budget must allow
constexpr int RW = 3 + QMAX + QMAX * QMAX;   // per-component result row in scratch
// Reading A16: T0 below the smallest normal double is an underflow (f_ij = 0): in gradual underflow
// the ratios E1/T0, E2/T0 have lost their precision (and 1/T0 overflows).
constexpr double TMIN = 2.2250738585072014e-308;

// Per-warp scratch for the per-pair setup (written redundantly by all lanes with identical
// values; every lane computes the same setup — SIMT issues it once per warp).
struct WarpScratch {
    double y[PMAX];
    double c[QMAX];
    double b[QMAX];
    double Sp[QMAX * QMAX];
    double ct[QMAX][QMAX];
    double St[QMAX][QMAX * QMAX];
    double Tk[QMAX];
    double Tkt[QMAX * QMAX];
    double phi[QMAX];
    double bc[QMAX];
    double Sc[QMAX * QMAX];
    double res[GMAX][RW];        // [logf (no prior), e1me2, e2, e3[q], e4[q*q]]
    double ll;
};

// ------------------------------------------------------------------------------------------
// SOV point loop for T_R (chi-normal form, reading R-T): this lane's share of
//   sum_l prod_k Phi(a_k(l)),  a_0 = s_l binv_0,  a_k = s_l binv_k - sum_{t<k} Cn_kt z_t,
//   z_t = Phi^{-1}(clamp(w_{l,t+1} e_t)).
// Per-q tuning of estep_cfust_kernel<Q> (measured on B200, profiles/r01_tuning.log; re-checked after
// the special-function refits, profiles/r01_retune.log: q = 3 with NP = 2 is 2.7 % faster on n = 3e5
// slices but 16 % slower at the full cfg5 size, so NP = 1 stays):
//   NP   lattice points per lane per loop iteration (independent SOV chains for the FP64 pipe),
//   MB   resident blocks per SM the register budget must allow (__launch_bounds__).
// CFUST_NP_Q<q> / CFUST_MB_Q<q> override them for experiment builds (scripts/build_variants.py).
#ifndef CFUST_NP_Q1
#define CFUST_NP_Q1 1
#endif
#ifndef CFUST_NP_Q2
#define CFUST_NP_Q2 1
#endif
#ifndef CFUST_NP_Q3
#define CFUST_NP_Q3 1
#endif
#ifndef CFUST_NP_Q4
#define CFUST_NP_Q4 2
#endif
#ifndef CFUST_NP_Q5
#define CFUST_NP_Q5 2
#endif
#ifndef CFUST_NP_Q6
#define CFUST_NP_Q6 2
#endif
#ifndef CFUST_MB_Q1
#define CFUST_MB_Q1 CFUST_MINB
#endif
#ifndef CFUST_MB_Q2
#define CFUST_MB_Q2 CFUST_MINB
#endif
#ifndef CFUST_MB_Q3
#define CFUST_MB_Q3 CFUST_MINB
#endif
#ifndef CFUST_MB_Q4
#define CFUST_MB_Q4 1
#endif
#ifndef CFUST_MB_Q5
#define CFUST_MB_Q5 1
#endif
#ifndef CFUST_MB_Q6
#define CFUST_MB_Q6 1
#endif
// CFUST_SOV_XT = q: the SOV loop of the q kernel takes exp from the 2^(j/64) table (exp_tab2).
// Off by default: measured at q = 3 (cfg5) -1.3 % E-step time for -12.6 % executed FP64 flops
// (the loop is latency bound: ncu `wait` ~2.9 per issue either way), q = 2 +1.3 %, q = 4 0
// (profiles/r02w_ab.log) — not worth a table load in every Phi.
#ifndef CFUST_SOV_XT
#define CFUST_SOV_XT 0
#endif
// CFUST_PF1_MASK bit q: the q kernel loads each point block's chi node / lattice coordinates one
// block ahead also with one warp per observation (SPLIT = 1; the SPLIT > 1 modes always do).  Same
// values in the same order: results are bitwise unchanged.  Measured (profiles/r02x_ab.log): q = 3
// (cfg5) -2.6 % E-step time, q = 4 (cfg2) -1.6 %, q = 2 +2.7 %, q = 6 +25 % (spills): profiles/r02z_ab.log.
#ifndef CFUST_PF1_MASK
#define CFUST_PF1_MASK ((1 << 3) | (1 << 4))
#endif
#ifndef CFUST_PFD_MASK
#define CFUST_PFD_MASK 0x7e   // the same one-point-ahead loads in sov_direct (SOV-direct estimator), q = 1..6: cfg5 -8.8 %, cfg2 -2.5 %, cfg4 -2.3 %, cfg1 -1 % (profiles/r02g2_ab_direct.log)
#endif
template <int Q>
struct Tune {
    static constexpr bool XT = Q == CFUST_SOV_XT;
    static constexpr bool PF = (CFUST_PF1_MASK >> Q) & 1;
    static constexpr int NP = Q == 1 ? CFUST_NP_Q1 : Q == 2 ? CFUST_NP_Q2 : Q == 3 ? CFUST_NP_Q3
                            : Q == 4 ? CFUST_NP_Q4 : Q == 5 ? CFUST_NP_Q5 : CFUST_NP_Q6;
    static constexpr int MB = Q == 1 ? CFUST_MB_Q1 : Q == 2 ? CFUST_MB_Q2 : Q == 3 ? CFUST_MB_Q3
                              : Q == 4 ? CFUST_MB_Q4 : Q == 5 ? CFUST_MB_Q5 : CFUST_MB_Q6;
};

// WT: also accumulate *wacc += f_l lv_l (exact e1, reading R2': lv = log V node table).
// SPLIT warps share one observation (small n): warp sub = wid % SPLIT takes the point blocks
// sub, sub + SPLIT, ... of 32 * NPTS points; split_sum combines the SPLIT warp totals.
template <int R, int NPTS, bool WT = false, int SPLIT = 1, bool XT = false, bool PF1 = false>
__device__ __forceinline__ double sov_lane_sum(const double (&binv)[R], const double (&Cn)[R * (R - 1) / 2],
                                               const double *__restrict__ chi, const double *__restrict__ W, int M,
                                               int lane, const double *__restrict__ lv = nullptr,
                                               double *wacc = nullptr) {
    // NPTS lattice points per iteration (l, l + 32, ...): independent chains for the FP64 pipe.
    // M is a power of two >= 1024, so 32 * NPTS * SPLIT divides it exactly (powers of two, <= 32).
    static_assert(NPTS == 1 || NPTS == 2 || NPTS == 4, "NPTS must divide M / 32");
    static_assert(NPTS * SPLIT <= 32, "32 * NPTS * SPLIT must divide M >= 1024");
    double acc[NPTS], accw[NPTS];
#pragma unroll
    for (int j = 0; j < NPTS; ++j) acc[j] = accw[j] = 0.0;
    const int sub = (SPLIT > 1) ? int(threadIdx.x >> 5) % SPLIT : 0;
    // Small-n (SPLIT) mode runs few warps per scheduler, so the L1 latency of each point's chi node
    // and lattice coordinates stalls the chain that consumes them: load one point block ahead.
    constexpr bool PF = SPLIT > 1 || PF1;
    constexpr int STEP = 32 * NPTS * SPLIT;
    double sn[NPTS], wn[NPTS][R > 1 ? R - 1 : 1];
    if constexpr (PF) {
        const int l1 = lane + sub * 32 * NPTS;
#pragma unroll
        for (int j = 0; j < NPTS; ++j) {
            sn[j] = __ldg(chi + l1 + 32 * j);
#pragma unroll
            for (int k = 1; k < R; ++k) wn[j][k - 1] = __ldg(W + k * M + l1 + 32 * j);
        }
    }
    for (int l0 = lane + sub * 32 * NPTS; l0 < M; l0 += STEP) {
        double s[NPTS], e[NPTS], f[NPTS], z[NPTS][R - 1], wv[NPTS][R > 1 ? R - 1 : 1];
        if constexpr (PF) {
            const int ln = (l0 + STEP < M) ? l0 + STEP : l0;   // (the last block re-reads its own points)
#pragma unroll
            for (int j = 0; j < NPTS; ++j) {
                s[j] = sn[j];
                sn[j] = __ldg(chi + ln + 32 * j);
#pragma unroll
                for (int k = 1; k < R; ++k) {
                    wv[j][k - 1] = wn[j][k - 1];
                    wn[j][k - 1] = __ldg(W + k * M + ln + 32 * j);
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < NPTS; ++j) {
                s[j] = __ldg(chi + l0 + 32 * j);
#pragma unroll
                for (int k = 1; k < R; ++k) wv[j][k - 1] = __ldg(W + k * M + l0 + 32 * j);   // lattice coordinate k (table)
            }
        }
#pragma unroll
        for (int j = 0; j < NPTS; ++j) {
            e[j] = Phi_t<XT>(s[j] * binv[0]);
            f[j] = e[j];
        }
#pragma unroll
        for (int k = 1; k < R; ++k) {
#pragma unroll
            for (int j = 0; j < NPTS; ++j) {
                const double w = wv[j][k - 1];
                double u = w * e[j];
                u = clamp_u(u, UMIN, UMAX);   // clamps (reading A15)
                z[j][k - 1] = Phiinv_t<XT>(u);
                double a = s[j] * binv[k];
#pragma unroll
                for (int t = 0; t < k; ++t) a -= Cn[(k * (k - 1)) / 2 + t] * z[j][t];
                e[j] = Phi_t<XT>(a);
                f[j] *= e[j];
            }
        }
#pragma unroll
        for (int j = 0; j < NPTS; ++j) {
            acc[j] += f[j];
            if constexpr (WT) accw[j] = fma(f[j], __ldg(lv + l0 + 32 * j), accw[j]);
        }
    }
    double tot = 0.0, totw = 0.0;
#pragma unroll
    for (int j = 0; j < NPTS; ++j) { tot += acc[j]; totw += accw[j]; }
    if constexpr (WT) *wacc = totw;
    return tot;
}

// Reordering (ascending b_k / sqrt(S_kk), stable; reading A13) and the scaled Cholesky factors of
// the SOV: binv_k = b_perm(k) / C_kk, Cn_kt = C_kt / C_kk.  false if S is not PD.
template <int R>
__device__ __forceinline__ bool sov_setup(const double *b, const double *S, int lds, double (&binv)[R],
                                          double (&Cn)[R * (R - 1) / 2]) {
    int perm[R];
    double key[R];
#pragma unroll
    for (int k = 0; k < R; ++k) { perm[k] = k; key[k] = b[k] / sqrt(S[k * lds + k]); }
    for (int i = 1; i < R; ++i) {
        const int pi = perm[i];
        int j = i - 1;
        while (j >= 0 && key[perm[j]] > key[pi]) { perm[j + 1] = perm[j]; --j; }
        perm[j + 1] = pi;
    }
    double C[R][R];
    for (int i = 0; i < R; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = S[perm[i] * lds + perm[j]];
            for (int k = 0; k < j; ++k) s -= C[i][k] * C[j][k];
            if (i == j) {
                if (!(s > 1e-300)) return false;
                C[i][i] = sqrt(s);
            } else {
                C[i][j] = s / C[j][j];
            }
        }
#pragma unroll
    for (int k = 0; k < R; ++k) binv[k] = b[perm[k]] / C[k][k];
#pragma unroll
    for (int k = 1; k < R; ++k)
#pragma unroll
        for (int t = 0; t < k; ++t) Cn[(k * (k - 1)) / 2 + t] = C[k][t] / C[k][k];
    return true;
}

// Sum of a warp-uniform value over the SPLIT warps of an observation group (named barrier 1 + group,
// fixed summation order: every warp of the group gets the same bits, so all take the same branches).
__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
template <int SPLIT>
__device__ __forceinline__ double split_sum(double v) {
    if constexpr (SPLIT == 1) {
        return v;
    } else {
        __shared__ double part[EW];
        const int wid = threadIdx.x >> 5, g0 = wid - wid % SPLIT, bar = 1 + wid / SPLIT;
        if ((threadIdx.x & 31) == 0) part[wid] = v;
        named_bar(bar, SPLIT * 32);
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < SPLIT; ++k) t += part[g0 + k];
        named_bar(bar, SPLIT * 32);   // the slots are reused by the next call
        return t;
    }
}

// T_R(b; 0, S, m): R = 0 -> 1; R = 1 -> univariate t CDF; R >= 2 -> lattice rule with
// univariate-prioritisation reordering (ascending b_k / sqrt(S_kk), stable; reading A13).
template <int R, int NP, int SPLIT = 1, bool XT = false, bool PF1 = false>
__device__ __noinline__ double T_eval(const double *b, const double *S, int lds, double m, double lbt,
                                      const double *__restrict__ chi, const double *__restrict__ W, int M,
                                      int lane) {
    if constexpr (R == 0) {
        return 1.0;
    } else if constexpr (R == 1) {
        return isinf(m) ? Phi(b[0] / sqrt(S[0])) : dev_t_cdf(b[0] / sqrt(S[0]), m, lbt);   // m = inf: normal family
    } else {
        double binv[R], Cn[R * (R - 1) / 2];
        if (!sov_setup<R>(b, S, lds, binv, Cn)) return CUDART_NAN;
        const double acc = sov_lane_sum<R, NP, false, SPLIT, XT, PF1>(binv, Cn, chi, W, M, lane);
        return split_sum<SPLIT>(warp_sum(acc)) / double(M);
    }
}

// NT >= 2 univariate T_1 values (T_eval<1> of argument arg = b / sqrt(S)) for one pair, one per
// lane (lane i < NT evaluates arg[i], the others repeat arg[0]) and broadcast: the warp-uniform
// continued fractions run side by side instead of one after another (q = 2: T_{q-1}, q = 3:
// T_{q-2}).  Bitwise the values T_eval<1> returns.
#ifndef CFUST_T1_LANES
#define CFUST_T1_LANES 1
#endif
template <int NT>
__device__ __forceinline__ void T1_lanes(const double *arg, double m, double lbt, int lane, double *out) {
    const int i = (lane < NT) ? lane : 0;
    const double x = arg[i];
    const double v = isinf(m) ? Phi(x) : dev_t_cdf(x, m, lbt);
#pragma unroll
    for (int k = 0; k < NT; ++k) out[k] = __shfl_sync(0xffffffffu, v, k);
}

// T_R on the lattice together with *wsum = (1/M) sum_l f_l lv_l over the same points (exact e1,
// reading R2'); R = 1 is evaluated on the lattice here too (f_l = Phi(s_l b / sqrt(S))).
template <int R, int NP, int SPLIT = 1, bool XT = false, bool PF1 = false>
__device__ __noinline__ double T_eval_w(const double *b, const double *S, int lds, const double *__restrict__ chi,
                                        const double *__restrict__ lv, const double *__restrict__ W, int M, int lane,
                                        double *wsum) {
    static_assert(R >= 1, "T_eval_w: R >= 1");
    double acc = 0.0, accw = 0.0;
    if constexpr (R == 1) {
        const double bs = b[0] / sqrt(S[0]);
        const int sub = (SPLIT > 1) ? int(threadIdx.x >> 5) % SPLIT : 0;
        for (int l = lane + 32 * sub; l < M; l += 32 * SPLIT) {
            const double f = Phi_t<XT>(__ldg(chi + l) * bs);
            acc += f;
            accw = fma(f, __ldg(lv + l), accw);
        }
    } else {
        double binv[R], Cn[R * (R - 1) / 2];
        if (!sov_setup<R>(b, S, lds, binv, Cn)) { *wsum = CUDART_NAN; return CUDART_NAN; }
        acc = sov_lane_sum<R, NP, true, SPLIT, XT, PF1>(binv, Cn, chi, W, M, lane, lv, &accw);
    }
    *wsum = split_sum<SPLIT>(warp_sum(accw)) / double(M);
    return split_sum<SPLIT>(warp_sum(acc)) / double(M);
}

// SOV-direct truncated moments (NEXT-3, reading D1): on T0's own SOV points, the last normal
// coordinate is drawn too (lattice coordinate Q), giving a posterior draw of (W, U) per point:
//   w = V/rho (1 for the skew-normal family), U = c - C xi / sqrt(w);  with weight f = prod e_k
// this lane's shares of  F = sum f, FW = sum f w, FL = sum f log w, F3 = sum f w U (permuted
// order), F4 = sum f w U U' (permuted, upper, packed) are returned warp-reduced in acc[].
// The first Q factors e_k are computed exactly as in sov_lane_sum, so T0 = F/M is bit-identical.
template <int Q>
__device__ __noinline__ bool sov_direct(const double *b, const double *S, int lds, const double *__restrict__ chi,
                                        const double *__restrict__ lv, const double *__restrict__ W, int M, int lane,
                                        double sqf, double m0r, double lrho, int sn, int (&perm)[Q], double *acc) {
    constexpr int NT = Q * (Q + 1) / 2;
    double key[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) { perm[k] = k; key[k] = b[k] / sqrt(S[k * lds + k]); }
    for (int i = 1; i < Q; ++i) {
        const int pi = perm[i];
        int j = i - 1;
        while (j >= 0 && key[perm[j]] > key[pi]) { perm[j + 1] = perm[j]; --j; }
        perm[j + 1] = pi;
    }
    double C[Q][Q];
    for (int i = 0; i < Q; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = S[perm[i] * lds + perm[j]];
            for (int k = 0; k < j; ++k) s -= C[i][k] * C[j][k];
            if (i == j) {
                if (!(s > 1e-300)) return false;
                C[i][i] = sqrt(s);
            } else {
                C[i][j] = s / C[j][j];
            }
        }
    double binv[Q], Cn[Q * (Q - 1) / 2 + 1], Cl[NT], cp[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) { binv[k] = b[perm[k]] / C[k][k]; cp[k] = b[perm[k]] / sqf; }
#pragma unroll
    for (int k = 1; k < Q; ++k)
#pragma unroll
        for (int t = 0; t < k; ++t) Cn[(k * (k - 1)) / 2 + t] = C[k][t] / C[k][k];
#pragma unroll
    for (int k = 0; k < Q; ++k)
#pragma unroll
        for (int t = 0; t <= k; ++t) Cl[(k * (k + 1)) / 2 + t] = C[k][t];
    double F = 0.0, FW = 0.0, FL = 0.0, F3[Q], F4[NT];
#pragma unroll
    for (int k = 0; k < Q; ++k) F3[k] = 0.0;
#pragma unroll
    for (int k = 0; k < NT; ++k) F4[k] = 0.0;
    // CFUST_PFD_MASK bit q: the chi node, lattice coordinates and log-V node of the next point are
    // loaded one point ahead of the chain that consumes them (as sov_lane_sum's PF; same values in
    // the same order, results bitwise unchanged).
    constexpr bool PFD = (CFUST_PFD_MASK >> Q) & 1;
    double sn1 = 0.0, lvn1 = 0.0, wn1[Q];
    if constexpr (PFD) {
        sn1 = __ldg(chi + lane);
        if (!sn) lvn1 = __ldg(lv + lane);
#pragma unroll
        for (int k = 0; k < Q; ++k) wn1[k] = __ldg(W + (k + 1) * M + lane);
    }
    for (int l = lane; l < M; l += 32) {
        double s, lvl = 0.0, wl[Q];
        if constexpr (PFD) {
            const int ln = (l + 32 < M) ? l + 32 : l;   // (the last point re-reads itself)
            s = sn1;
            sn1 = __ldg(chi + ln);
            lvl = lvn1;
            if (!sn) lvn1 = __ldg(lv + ln);
#pragma unroll
            for (int k = 0; k < Q; ++k) { wl[k] = wn1[k]; wn1[k] = __ldg(W + (k + 1) * M + ln); }
        } else {
            s = __ldg(chi + l);
        }
        double e = Phi(s * binv[0]);
        double f = e;
        double xi[Q];
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            if (k > 0) {
                double a = s * binv[k];
#pragma unroll
                for (int t = 0; t < k; ++t) a -= Cn[(k * (k - 1)) / 2 + t] * xi[t];
                e = Phi(a);
                f *= e;
            }
            double u = (PFD ? wl[k] : __ldg(W + (k + 1) * M + l)) * e;
            u = clamp_u(u, UMIN, UMAX);
            xi[k] = Phiinv(u);
        }
        const double w = sn ? 1.0 : m0r * s * s;
        const double isw = sn ? 1.0 : div_fast(1.0, s * sqf);   // 1 / sqrt(w)
        const double fw = f * w;
        F += f;
        FW += fw;
        if (!sn) FL = fma(f, (PFD ? lvl : __ldg(lv + l)) - lrho, FL);
        double U[Q];
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            double z = 0.0;
#pragma unroll
            for (int t = 0; t <= k; ++t) z = fma(Cl[(k * (k + 1)) / 2 + t], xi[t], z);
            U[k] = cp[k] - z * isw;
            F3[k] = fma(fw, U[k], F3[k]);
        }
#pragma unroll
        for (int a = 0; a < Q; ++a)
#pragma unroll
            for (int bb = a; bb < Q; ++bb) F4[a * Q - a * (a - 1) / 2 + (bb - a)] = fma(fw * U[a], U[bb], F4[a * Q - a * (a - 1) / 2 + (bb - a)]);
    }
    acc[0] = warp_sum(F);
    acc[1] = warp_sum(FW);
    acc[2] = warp_sum(FL);
#pragma unroll
    for (int k = 0; k < Q; ++k) acc[3 + k] = warp_sum(F3[k]);
#pragma unroll
    for (int k = 0; k < NT; ++k) acc[3 + Q + k] = warp_sum(F4[k]);
    return true;
}

template <int Q>
__device__ void pair_eval_direct(const CompDev &cp, int p, const double *__restrict__ W, int M,
                                 const double *__restrict__ chi, WarpScratch &ws, double *res, int lane, int family) {
    const bool nrm = family == 1;
    double r[PMAX], v[PMAX];
    double d = 0.0;
#pragma unroll
    for (int a = 0; a < PMAX; ++a) {
        if (a < p) {
            r[a] = ws.y[a] - cp.mu[a];
            double s = r[a];
#pragma unroll
            for (int bb = 0; bb < a; ++bb) s -= cp.L[a * PMAX + bb] * v[bb];
            v[a] = s * cp.Linv[a];
            d += v[a] * v[a];
        }
    }
    const double nu = cp.nu, m0 = cp.m0, rho = nu + d;
    const double logt = nrm ? cp.kappa - 0.5 * d : cp.kappa - 0.5 * m0 * log1p(d / nu);
    const double sqf = nrm ? 1.0 : sqrt(m0 / rho);
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < PMAX; ++a)
            if (a < p) s += cp.A[k * PMAX + a] * r[a];
        ws.b[k] = s * sqf;
    }
    constexpr int NT = Q * (Q + 1) / 2;
    double acc[3 + Q + NT];
    int perm[Q];
    const bool ok = sov_direct<Q>(ws.b, cp.Lam, QMAX, chi, chi + CHI_LV * M, W, M, lane, sqf, nrm ? 0.0 : m0 / rho,
                                  log(rho), family, perm, acc);
    const double F = ok ? acc[0] : 0.0;
    double T0 = F / double(M);
    if (Q == 1) T0 = T_eval<1, 1>(ws.b, cp.Lam, QMAX, nrm ? CUDART_INF : m0, cp.lbt[0], chi, W, M, lane);   // exact T_1
    const double e1me2_a5 = nrm ? 0.0 : cp.psi_half_m0 - log(0.5 * rho) - m0 / rho;
    if (!(T0 >= TMIN) || !(F > 0.0)) {   // reading A16
        res[0] = -CUDART_INF;
        res[1] = e1me2_a5;
        for (int k = 2; k < 3 + Q + Q * Q; ++k) res[k] = 0.0;
        return;
    }
    // ratios by IEEE division (F may be subnormal)
    res[0] = Q * CUDART_LN2 + logt + log(T0);
    res[2] = acc[1] / F;
    res[1] = nrm ? 0.0 : acc[2] / F - res[2];
#pragma unroll
    for (int k = 0; k < Q; ++k) res[3 + perm[k]] = acc[3 + k] / F;
#pragma unroll
    for (int a = 0; a < Q; ++a)
#pragma unroll
        for (int bb = a; bb < Q; ++bb) {
            const double val = acc[3 + Q + a * Q - a * (a - 1) / 2 + (bb - a)] / F;
            res[3 + Q + perm[a] * Q + perm[bb]] = val;
            res[3 + Q + perm[bb] * Q + perm[a]] = val;
        }
}

// Per pair (observation in ws.y, component cp): O2-O8 of DESIGN.md §3.
// MODE 1 computes only log f (T0).  Results go to res[] (identical in all lanes).
template <int Q, int MODE, int SPLIT = 1>
__device__ void pair_eval(const CompDev &cp, int p, const double *__restrict__ W, int M, const double *__restrict__ chi,
                          WarpScratch &ws, double *res, int lane, int e1_exact, int family) {
    // family 1 = skew-normal (CFUSN, nu = inf; reading F1): W = 1, normal SOV (radius nodes = 1),
    // normal densities and conditionals; every t-specific factor below becomes 1.
    const bool nrm = family == 1;
    double r[PMAX], v[PMAX];
    double d = 0.0;
#pragma unroll
    for (int a = 0; a < PMAX; ++a) {
        if (a < p) {
            r[a] = ws.y[a] - cp.mu[a];
            double s = r[a];
#pragma unroll
            for (int bb = 0; bb < a; ++bb) s -= cp.L[a * PMAX + bb] * v[bb];
            v[a] = s * cp.Linv[a];
            d += v[a] * v[a];
        }
    }
    const double nu = cp.nu, m0 = cp.m0, rho = nu + d;
    const double logt = nrm ? cp.kappa - 0.5 * d : cp.kappa - 0.5 * m0 * log1p(d / nu);
    const double mT0 = nrm ? CUDART_INF : m0;   // df of T0 (inf: normal)
    double c[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < PMAX; ++a)
            if (a < p) s += cp.A[k * PMAX + a] * r[a];
        c[k] = s;
    }
    // T0 (density, Eq. (2)) and T2 (for e2)
    const double sq0 = nrm ? 1.0 : sqrt(m0 / rho);
#pragma unroll
    for (int k = 0; k < Q; ++k) ws.b[k] = c[k] * sq0;
    double T0, e1x = 0.0;
    if (MODE != 1 && e1_exact) {   // exact e1 = (sum f lv)/(sum f) - log rho on T0's points (R2')
        double wsum;
        const double T0lat = T_eval_w<Q, Tune<Q>::NP, SPLIT, Tune<Q>::XT, Tune<Q>::PF>(ws.b, cp.Lam, QMAX, chi, chi + CHI_LV * M, W, M, lane, &wsum);
        T0 = (Q == 1) ? T_eval<1, 1>(ws.b, cp.Lam, QMAX, m0, cp.lbt[0], chi, W, M, lane) : T0lat;   // density: exact T_1
        e1x = wsum / T0lat - log(rho);
    } else {
        T0 = T_eval<Q, Tune<Q>::NP, SPLIT, Tune<Q>::XT, Tune<Q>::PF>(ws.b, cp.Lam, QMAX, mT0, cp.lbt[0], chi, W, M, lane);
    }
    if (MODE == 1) {
        res[0] = (T0 >= TMIN) ? Q * CUDART_LN2 + logt + log(T0) : -CUDART_INF;
        return;
    }
    double T2 = T0;   // normal family: E1 = c P + Lambda h uses P = T0, and e2 = 1
    if (!nrm) {
        const double sq2 = sqrt((m0 + 2.0) / rho);
#pragma unroll
        for (int k = 0; k < Q; ++k) ws.b[k] = c[k] * sq2;
        T2 = T_eval<Q, Tune<Q>::NP, SPLIT, Tune<Q>::XT, Tune<Q>::PF>(ws.b, cp.Lam, QMAX, m0 + 2.0, cp.lbt[2], chi + CHI_M2 * M, W, M, lane);
    }
    res[1] = nrm ? 0.0 : cp.psi_half_m0 - log(0.5 * rho) - m0 / rho;      // e1 - e2, reading A5
    if (!(T0 >= TMIN)) {                                        // reading A16
        res[0] = -CUDART_INF;
        for (int k = 2; k < 3 + Q + Q * Q; ++k) res[k] = 0.0;
        return;
    }
    // S' = (rho/m0) Lambda  (normal: Lambda)
    const double sc = nrm ? 1.0 : rho / m0;
#pragma unroll
    for (int k = 0; k < Q; ++k)
#pragma unroll
        for (int l = 0; l < Q; ++l) ws.Sp[k * QMAX + l] = sc * cp.Lam[k * QMAX + l];
    const double *Sp = ws.Sp;
    // phi_k = t_1(0; c_k, S'_kk, m0) and conditionals on x_k = 0 (df m0 + 1)
    constexpr int Q1 = Q - 1;
    constexpr int Q2 = (Q >= 2) ? Q - 2 : 0;
    for (int k = 0; k < Q; ++k) {
        const double skk = Sp[k * QMAX + k];
        ws.phi[k] = exp(nrm ? dev_n1_logpdf0(c[k], skk) : dev_t1_logpdf0(c[k], skk, m0, cp.lgc_m0));
        if constexpr (Q >= 2) {
            const double fac = nrm ? 1.0 : (m0 + c[k] * c[k] / skk) / (m0 + 1.0);
            int ia = 0;
            for (int i = 0; i < Q; ++i) {
                if (i == k) continue;
                ws.ct[k][ia] = c[i] - Sp[i * QMAX + k] * c[k] / skk;
                int ib = 0;
                for (int j = 0; j < Q; ++j) {
                    if (j == k) continue;
                    ws.St[k][ia * QMAX + ib] = fac * (Sp[i * QMAX + j] - Sp[i * QMAX + k] * Sp[k * QMAX + j] / skk);
                    ++ib;
                }
                ++ia;
            }
        }
    }
    const double rat = nrm ? 1.0 : (m0 + 1.0) / (m0 - 1.0);   // S~' = rat * S~ (df m0 - 1)
    // T_{q-2} for each pair {k < t}: condition t_{q-1}(c~(k), S~'(k), m0-1) on x_t = 0 (df m0)
    if constexpr (Q >= 3) {
        for (int k = 0; k < Q; ++k)
            for (int t = k + 1; t < Q; ++t) {
                const int at = t - 1;                  // position of t among "others of k" (t > k)
                const double saa = rat * ws.St[k][at * QMAX + at];
                const double cta = ws.ct[k][at];
                const double fac2 = nrm ? 1.0 : (m0 - 1.0 + cta * cta / saa) / m0;
                int ib = 0;
                for (int i = 0; i < Q1; ++i) {
                    if (i == at) continue;
                    const double sia = rat * ws.St[k][i * QMAX + at];
                    ws.bc[ib] = ws.ct[k][i] - sia * cta / saa;
                    int jb = 0;
                    for (int j = 0; j < Q1; ++j) {
                        if (j == at) continue;
                        const double sij = rat * ws.St[k][i * QMAX + j];
                        const double saj = rat * ws.St[k][at * QMAX + j];
                        ws.Sc[ib * QMAX + jb] = fac2 * (sij - sia * saj / saa);
                        ++jb;
                    }
                    ++ib;
                }
                if constexpr (Q2 == 1 && CFUST_T1_LANES) {
                    ws.Tkt[t * QMAX + k] = ws.bc[0] / sqrt(ws.Sc[0]);   // T_1 argument, evaluated below
                } else {
                    const double val = T_eval<Q2, Tune<Q>::NP, SPLIT, Tune<Q>::XT, Tune<Q>::PF>(ws.bc, ws.Sc, QMAX, mT0, cp.lbt[0], chi, W, M, lane);
                    ws.Tkt[k * QMAX + t] = val;
                    ws.Tkt[t * QMAX + k] = val;            // symmetric in {k, t} (A17)
                }
            }
        if constexpr (Q2 == 1 && CFUST_T1_LANES) {   // q = 3: the three T_1 side by side; arguments at (t, k), t > k
            __syncwarp();
            const double arg[3] = {ws.Tkt[1 * QMAX + 0], ws.Tkt[2 * QMAX + 0], ws.Tkt[2 * QMAX + 1]};
            double val[3];
            T1_lanes<3>(arg, mT0, cp.lbt[0], lane, val);
            __syncwarp();
            ws.Tkt[0 * QMAX + 1] = ws.Tkt[1 * QMAX + 0] = val[0];
            ws.Tkt[0 * QMAX + 2] = ws.Tkt[2 * QMAX + 0] = val[1];
            ws.Tkt[1 * QMAX + 2] = ws.Tkt[2 * QMAX + 1] = val[2];
            __syncwarp();
        }
    }
    // T_{q-1}(c~(k); 0, S~(k), m0+1) and h_k = phi_k T~(k)
    double h[Q];
    if constexpr (Q1 == 1 && CFUST_T1_LANES) {   // q = 2: both T_1 side by side
        const double arg[2] = {ws.ct[0][0] / sqrt(ws.St[0][0]), ws.ct[1][0] / sqrt(ws.St[1][0])};
        double tk[2];
        T1_lanes<2>(arg, nrm ? CUDART_INF : m0 + 1.0, cp.lbt[1], lane, tk);
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            ws.Tk[k] = tk[k];
            h[k] = ws.phi[k] * tk[k];
        }
    } else {
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            double tk = 1.0;
            if constexpr (Q >= 2)
                tk = T_eval<Q1, Tune<Q>::NP, SPLIT, Tune<Q>::XT, Tune<Q>::PF>(ws.ct[k], ws.St[k], QMAX, nrm ? CUDART_INF : m0 + 1.0, cp.lbt[1], chi + CHI_M1 * M, W, M, lane);
            ws.Tk[k] = tk;
            h[k] = ws.phi[k] * tk;
        }
    }
    // E1 = c T2 + S' h
    double E1[Q];
#pragma unroll
    for (int a = 0; a < Q; ++a) {
        double s = c[a] * T2;
#pragma unroll
        for (int k = 0; k < Q; ++k) s += Sp[a * QMAX + k] * h[k];
        E1[a] = s;
    }
    // G_kl = phi_k [ c~(k)_l T~(k) + (S~'(k) h(k))_l ],  h(k)_t = t_1(0; c~_t, S~'_tt, m0-1) T(k,t)
    double G[Q][Q];
#pragma unroll
    for (int k = 0; k < Q; ++k)
#pragma unroll
        for (int l = 0; l < Q; ++l) G[k][l] = 0.0;
    if constexpr (Q >= 2) {
        for (int k = 0; k < Q; ++k) {
            double hk[QMAX];
            for (int a = 0; a < Q1; ++a) {
                const int t = (a < k) ? a : a + 1;
                const double saa = rat * ws.St[k][a * QMAX + a];
                const double tkt = (Q >= 3) ? ws.Tkt[k * QMAX + t] : 1.0;
                hk[a] = exp(nrm ? dev_n1_logpdf0(ws.ct[k][a], saa) : dev_t1_logpdf0(ws.ct[k][a], saa, m0 - 1.0, cp.lgc_m0m1)) * tkt;
            }
            for (int a = 0; a < Q1; ++a) {
                const int l = (a < k) ? a : a + 1;
                double s = ws.ct[k][a] * ws.Tk[k];
                for (int bb = 0; bb < Q1; ++bb) s += rat * ws.St[k][a * QMAX + bb] * hk[bb];
                G[k][l] = ws.phi[k] * s;
            }
        }
    }
    // E2 = sym( S'(G + T0 I) + c E1' );  e2, e3, e4 (O8)
    const double fr = nrm ? 1.0 : m0 / rho;
    // T0 >= DBL_MIN here (reading A16 above), so 1/T0 is finite
    const double inv = 1.0 / T0;
    res[0] = Q * CUDART_LN2 + logt + log(T0);
    res[2] = nrm ? 1.0 : fr * T2 * inv;
    if (e1_exact) res[1] = e1x - res[2];
#pragma unroll
    for (int a = 0; a < Q; ++a) res[3 + a] = fr * E1[a] * inv;
    double E2[Q][Q];
#pragma unroll
    for (int a = 0; a < Q; ++a)
#pragma unroll
        for (int bb = 0; bb < Q; ++bb) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < Q; ++k) s += Sp[a * QMAX + k] * (G[k][bb] + (k == bb ? T0 : 0.0));
            E2[a][bb] = s + c[a] * E1[bb];
        }
#pragma unroll
    for (int a = 0; a < Q; ++a)
#pragma unroll
        for (int bb = 0; bb < Q; ++bb) res[3 + Q + a * Q + bb] = fr * 0.5 * (E2[a][bb] + E2[bb][a]) * inv;
}

// Stats entry decode: code = type | i << 4 | a << 8 | b << 12
enum : int { ST_S0 = 0, ST_S1, ST_S2, ST_S3, ST_S4, ST_S5, ST_S6, ST_S7 };

__device__ inline int stat_code(int e, int p, int q, int K) {
    const int i = e / K;
    int k = e % K;
    int type, a = 0, b = 0;
    if (k == 0) type = ST_S0;
    else if (k == 1) type = ST_S1;
    else if ((k -= 2) < p) { type = ST_S2; a = k; }
    else if ((k -= p) < p * (p + 1) / 2) {
        type = ST_S3;
        int row = 0;
        while (k >= p - row) { k -= p - row; ++row; }
        a = row; b = row + k;
    } else if ((k -= p * (p + 1) / 2) < q) { type = ST_S4; a = k; }
    else if ((k -= q) < q * (q + 1) / 2) {
        type = ST_S5;
        int row = 0;
        while (k >= q - row) { k -= q - row; ++row; }
        a = row; b = row + k;
    } else if ((k -= q * (q + 1) / 2) < p * q) { type = ST_S6; a = k / q; b = k % q; }
    else type = ST_S7;
    return type | (i << 4) | (a << 8) | (b << 12);
}

struct EArgs {
    const double *__restrict__ y;
    int64_t n;
    int p, g, K;
    const CompDev *__restrict__ comp;
    const double *__restrict__ chi;
    const double *__restrict__ W;   // [q][M] lattice coordinates w_{l,k}
    int M;
    double *__restrict__ partials;
    int *status;
    const int64_t *__restrict__ idx;
    int64_t cnt;
    double *__restrict__ pair_out;
    int e1_exact;                   // 1: exact e1 (reading R2'), 0: reading A5
    int family;                     // 0 skew-t (CFUST), 1 skew-normal (CFUSN; q = 0: Gaussian)
    int direct;                     // 1: SOV-direct truncated moments (reading D1)
    double *__restrict__ tau_out;   // MODE 1: tau [n][g] (NULL: log-likelihood only)
    int32_t *__restrict__ label_out;   // MODE 1: MAP component per observation
};

// MODE 0: E-step statistics; 1: log-likelihood only; 2: per-pair dump of idx[0..cnt).
// DIRECT: SOV-direct truncated moments (reading D1) — a separate instantiation, so the analytic
// kernel's register allocation is not burdened by the direct path.
#ifndef CFUST_MBD
#define CFUST_MBD 2   // resident blocks/SM for the SOV-direct instantiations (profiles/r01_direct_tuning.log)
#endif
// SPLIT > 1 (analytic statistics and density passes, small n): SPLIT warps per observation, each on 1/SPLIT of the
// lattice points (sov_lane_sum), totals combined per integral (split_sum); warp 0 of the group
// accumulates.  The per-pair setup is repeated by the SPLIT warps (identical inputs and bits).
template <int Q, int MODE, bool DIRECT = false, int SPLIT = 1>
__global__ void __launch_bounds__(EW * 32, (DIRECT && CFUST_MBD > 0) ? CFUST_MBD : Tune<Q>::MB) estep_cfust_kernel(EArgs A) {
    static_assert(SPLIT == 1 || (!DIRECT && MODE != 2 && EW % SPLIT == 0), "SPLIT: analytic statistics / density pass only");
    constexpr int OPB = EW / SPLIT;   // observations per block per sweep
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int p = A.p, g = A.g, K = A.K, GK = g * K;
    CompDev *comp = reinterpret_cast<CompDev *>(smem_raw);
    WarpScratch *wsa = reinterpret_cast<WarpScratch *>(comp + g);
    double *acc_all = reinterpret_cast<double *>(wsa + EW);          // [EW][GK + 1]
    int *codes = reinterpret_cast<int *>(acc_all + EW * (GK + 1));   // [GK]
    for (int t = threadIdx.x; t < g * int(sizeof(CompDev) / sizeof(double)); t += blockDim.x)
        reinterpret_cast<double *>(comp)[t] = reinterpret_cast<const double *>(A.comp)[t];
    for (int e = threadIdx.x; e < GK; e += blockDim.x) codes[e] = stat_code(e, p, Q, K);
    for (int e = threadIdx.x; e < EW * (GK + 1); e += blockDim.x) acc_all[e] = 0.0;
    __syncthreads();
    WarpScratch &ws = wsa[wid];
    double *acc = acc_all + wid * (GK + 1);
    const int M = A.M;
    const int64_t ngroups = int64_t(gridDim.x) * OPB;
    const int64_t total = (MODE == 2) ? A.cnt : A.n;
    const bool lead = (SPLIT == 1) || (wid % SPLIT == 0);   // the warp that accumulates for its group
    double ll = 0.0;
    for (int64_t jj = int64_t(blockIdx.x) * OPB + wid / SPLIT; jj < total; jj += ngroups) {
        const int64_t j = (MODE == 2) ? A.idx[jj] : jj;
        __syncwarp();
        if (lane < p) ws.y[lane] = A.y[j * p + lane];
        __syncwarp();
        for (int i = 0; i < g; ++i)
        {
            const double *chi_i = A.chi + size_t(i) * CHI_ROWS * M;
            if constexpr (DIRECT && MODE != 1)
                pair_eval_direct<Q>(comp[i], p, A.W, M, chi_i, ws, ws.res[i], lane, A.family);
            else
                pair_eval<Q, MODE == 1 ? 1 : 0, SPLIT>(comp[i], p, A.W, M, chi_i, ws, ws.res[i], lane, A.e1_exact, A.family);
        }
        __syncwarp();
        // Eq. (3)-(4): LSE over components, tau
        double lf[GMAX], mx = -CUDART_INF;
#pragma unroll
        for (int i = 0; i < GMAX; ++i)
            if (i < g) { lf[i] = comp[i].logpi + ws.res[i][0]; mx = fmax(mx, lf[i]); }
        if (mx == -CUDART_INF) {
            if (lane == 0 && lead) atomicOr(A.status, 1);
            continue;
        }
        double se = 0.0;
#pragma unroll
        for (int i = 0; i < GMAX; ++i)
            if (i < g) se += exp(lf[i] - mx);
        const double lse = mx + log(se);
        if (lead) ll += lse;
        if constexpr (MODE == 1) {
            if (A.tau_out && lane == 0 && lead) {   // responsibilities and the MAP label (ties -> lowest index)
                int best = 0;
                for (int i = 0; i < g; ++i) {
                    A.tau_out[size_t(j) * g + i] = exp(lf[i] - lse);
                    if (lf[i] > lf[best]) best = i;
                }
                A.label_out[j] = best;
            }
            continue;
        }
        double tau[GMAX];
#pragma unroll
        for (int i = 0; i < GMAX; ++i) tau[i] = (i < g) ? exp(lf[i] - lse) : 0.0;
        if constexpr (MODE == 2) {
            const int PWo = 4 + Q + Q * Q;
            double *o = A.pair_out + size_t(jj) * g * PWo;
            for (int e = lane; e < g * PWo; e += 32) {
                const int i = e / PWo, k = e % PWo;
                double lfi = 0.0, ti = 0.0;
#pragma unroll
                for (int c2 = 0; c2 < GMAX; ++c2)
                    if (c2 == i) { lfi = lf[c2]; ti = tau[c2]; }
                o[e] = (k == 0) ? lfi : (k == 1) ? ti : ws.res[i][k - 1];
            }
            continue;
        }
        // accumulate the eight sufficient statistics (reading A4); lane-owned entries
        if (!lead) continue;
        for (int e = lane; e < GK; e += 32) {
            const int code = codes[e];
            const int type = code & 15, i = (code >> 4) & 15, a = (code >> 8) & 15, bq = (code >> 12) & 15;
            double ti = 0.0;
#pragma unroll
            for (int c2 = 0; c2 < GMAX; ++c2)
                if (c2 == i) ti = tau[c2];
            if (!(ti > 0.0)) continue;
            const double *rs = ws.res[i];
            double val;
            switch (type) {
                case ST_S0: val = 1.0; break;
                case ST_S1: val = rs[2]; break;
                case ST_S2: val = rs[2] * ws.y[a]; break;
                case ST_S3: val = rs[2] * ws.y[a] * ws.y[bq]; break;
                case ST_S4: val = rs[3 + a]; break;
                case ST_S5: val = rs[3 + Q + a * Q + bq]; break;
                case ST_S6: val = ws.y[a] * rs[3 + bq]; break;
                default: val = rs[1]; break;
            }
            acc[e] += ti * val;
        }
    }
    if (MODE == 2) return;
    if (lane == 0) acc[GK] = ll;
    __syncthreads();
    double *out = A.partials + size_t(blockIdx.x) * (GK + 1);
    for (int e = threadIdx.x; e <= GK; e += blockDim.x) {
        double s = 0.0;
        for (int w = 0; w < EW; ++w) s += acc_all[w * (GK + 1) + e];
        out[e] = s;
    }
}

// ------------------------------------------------------------------------------------------
// q == 0: t-mixture E-step (Delta = 0), streaming y from HBM.
// Tile = TT observations = TT threads.  Phase 1: thread per observation evaluates all g
// components (d, log f, tau, e2, e1-e2) and writes y (augmented with a constant 1) and the
// weights tau*e2, tau, tau*(e1-e2) to shared memory.  Phase 2: the tile contraction
//   S1/S2/S3_i += sum_j (tau e2)_ij y~_j y~_j'   (y~ = (y, 1): S3 = upper block, S2 = last column,
//                                                 S1 = corner),   S0_i, S7_i = weighted row sums,
// split into register-blocked 3x3 tasks x TCH row-chunks; every thread keeps its two tasks'
// accumulators in registers across tiles.  Deterministic: fixed task/chunk/row order.
// (A product-per-lane variant with broadcast weights measured 1.8x slower: idle lanes, 8 warps/SM.)
constexpr int TT = 256;    // observations per tile (= threads per block)
constexpr int TCH = 8;     // row chunks per contraction task (rows r = rr*TCH + ch: bank-spread)
constexpr int TSLOT = 2;   // contraction (task, chunk) slots per thread

template <int P>
struct TLayout {
    static constexpr int PE = P + 1;               // y~ = (y, 1)
    static constexpr int NB = (PE + 2) / 3;        // 3-wide coordinate blocks
    static constexpr int YS = 3 * NB;              // row stride of y~ in smem (zero padded)
    static constexpr int NBP = NB * (NB + 1) / 2;  // upper block pairs (A <= B)
    static constexpr int WS = GMAX + 1;            // row stride of the weight arrays (bank spread)
};

static_assert(GMAX * (TLayout<PMAX>::NBP + 1) * TCH <= TSLOT * TT, "contraction tasks exceed thread slots");

template <int P>
__global__ void __launch_bounds__(TT, 2) estep_t_kernel(EArgs A, int mode) {
    using Lt = TLayout<P>;
    constexpr int NB = Lt::NB, YS = Lt::YS, NBP = Lt::NBP, WS = Lt::WS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int g = A.g, K = A.K, GK = g * K;
    CompDev *comp = reinterpret_cast<CompDev *>(smem_raw);
    double *yt = reinterpret_cast<double *>(comp + g);   // [TT][YS]
    double *we = yt + TT * YS;                           // [TT][WS] tau*e2
    double *wt = we + TT * WS;                           // [TT][WS] tau
    double *wl = wt + TT * WS;                           // [TT][WS] tau*(e1-e2)
    double *red = wl + TT * WS;                          // end-of-kernel reduction scratch
    for (int k = t; k < g * int(sizeof(CompDev) / sizeof(double)); k += TT)
        reinterpret_cast<double *>(comp)[k] = reinterpret_cast<const double *>(A.comp)[k];
    __syncthreads();
    const int ntask = g * (NBP + 1);   // per component: NBP block pairs + 1 scalar task (S0, S7)
    double acc[TSLOT][9];
#pragma unroll
    for (int sl = 0; sl < TSLOT; ++sl)
#pragma unroll
        for (int k = 0; k < 9; ++k) acc[sl][k] = 0.0;
    double ll = 0.0;
    const int64_t n = A.n;
    const int64_t ntiles = (n + TT - 1) / TT;
    for (int64_t tb = blockIdx.x; tb < ntiles; tb += gridDim.x) {
        // ---------------- phase 1: one observation per thread, all components
        const int64_t j = tb * TT + t;
        double y[P];
        const bool valid = j < n;
        if (valid) {
            const double *yr = A.y + j * P;
            if constexpr (P % 2 == 0) {
#pragma unroll
                for (int a = 0; a < P; a += 2) {
                    const double2 v2 = __ldg(reinterpret_cast<const double2 *>(yr + a));
                    y[a] = v2.x;
                    y[a + 1] = v2.y;
                }
            } else {
#pragma unroll
                for (int a = 0; a < P; ++a) y[a] = __ldg(yr + a);
            }
        } else {
#pragma unroll
            for (int a = 0; a < P; ++a) y[a] = 0.0;
        }
        double lf[GMAX], l1[GMAX], dd[GMAX];
        double mx = -CUDART_INF;
#pragma unroll
        for (int i = 0; i < GMAX; ++i) {
            if (i < g) {
                const CompDev &cp = comp[i];
                double v[P], d = 0.0;
#pragma unroll
                for (int a = 0; a < P; ++a) {
                    double s = y[a] - cp.mu[a];
#pragma unroll
                    for (int b = 0; b < a; ++b) s -= cp.L[a * PMAX + b] * v[b];
                    v[a] = s * cp.Linv[a];
                    d += v[a] * v[a];
                }
                dd[i] = d;
                l1[i] = (A.family == 1) ? 0.0 : log1p(d * cp.inv_nu);
                lf[i] = cp.logpi + cp.kappa - ((A.family == 1) ? 0.5 * d : 0.5 * cp.m0 * l1[i]);
                mx = fmax(mx, lf[i]);
            }
        }
        double se = 0.0;
#pragma unroll
        for (int i = 0; i < GMAX; ++i)
            if (i < g) { lf[i] = exp(lf[i] - mx); se += lf[i]; }   // lf now holds exp(lf - max)
        if (valid && mx == -CUDART_INF) atomicOr(A.status, 1);
        if (valid) ll += mx + log(se);
        if (mode == 1) continue;
        const double ise = 1.0 / se;
#pragma unroll
        for (int a = 0; a < YS; ++a) yt[t * YS + a] = (a < P) ? y[a] : (a == P ? 1.0 : 0.0);
#pragma unroll
        for (int i = 0; i < GMAX; ++i) {
            if (i < g) {
                const CompDev &cp = comp[i];
                const double tau = valid ? lf[i] * ise : 0.0;
                const double e2 = (A.family == 1) ? 1.0 : cp.m0 / (cp.nu + dd[i]);
                const double e1me2 = (A.family == 1) ? 0.0 : cp.psi_half_m0 - (cp.log_half_nu + l1[i]) - e2;
                we[t * WS + i] = tau * e2;
                wt[t * WS + i] = tau;
                wl[t * WS + i] = tau * e1me2;
            }
        }
        __syncthreads();
        // ---------------- phase 2: tile contraction (register-blocked 3x3 tasks)
#pragma unroll
        for (int sl = 0; sl < TSLOT; ++sl) {
            const int ts = t + sl * TT;
            if (ts < ntask * TCH) {
                const int task = ts / TCH, ch = ts % TCH;
                const int i = task / (NBP + 1), kind = task % (NBP + 1);
                if (kind == NBP) {   // S0 = sum tau, S7 = sum tau (e1 - e2)
                    for (int rr = 0; rr < TT / TCH; ++rr) {
                        const int r = rr * TCH + ch;
                        acc[sl][0] += wt[r * WS + i];
                        acc[sl][1] += wl[r * WS + i];
                    }
                } else {
                    int BA = 0, rem = kind;
                    while (rem >= NB - BA) { rem -= NB - BA; ++BA; }
                    const int BB = BA + rem;
                    for (int rr = 0; rr < TT / TCH; ++rr) {
                        const int r = rr * TCH + ch;
                        const double w = we[r * WS + i];
                        const double *yr = yt + r * YS;
                        const double ya0 = w * yr[3 * BA], ya1 = w * yr[3 * BA + 1], ya2 = w * yr[3 * BA + 2];
                        const double yb0 = yr[3 * BB], yb1 = yr[3 * BB + 1], yb2 = yr[3 * BB + 2];
                        acc[sl][0] += ya0 * yb0; acc[sl][1] += ya0 * yb1; acc[sl][2] += ya0 * yb2;
                        acc[sl][3] += ya1 * yb0; acc[sl][4] += ya1 * yb1; acc[sl][5] += ya1 * yb2;
                        acc[sl][6] += ya2 * yb0; acc[sl][7] += ya2 * yb1; acc[sl][8] += ya2 * yb2;
                    }
                }
            }
        }
        __syncthreads();
    }
    // ---------------- block reduction: log-likelihood
    ll = warp_sum(ll);
    __syncthreads();
    if (lane == 0) red[wid] = ll;
    __syncthreads();
    double *out = A.partials + size_t(blockIdx.x) * (GK + 1);
    if (t == 0) {
        double s = 0.0;
        for (int w = 0; w < TT / 32; ++w) s += red[w];
        out[GK] = s;
    }
    if (mode == 1) return;
    __syncthreads();
    // task accumulators -> smem [ntask][TCH][9], then per statistics entry in chunk order
    double *tr = red + 32;
#pragma unroll
    for (int sl = 0; sl < TSLOT; ++sl) {
        const int ts = t + sl * TT;
        if (ts < ntask * TCH)
#pragma unroll
            for (int k = 0; k < 9; ++k) tr[ts * 9 + k] = acc[sl][k];
    }
    __syncthreads();
    auto task_sum = [&](int task, int k) {
        double s = 0.0;
        for (int ch = 0; ch < TCH; ++ch) s += tr[(task * TCH + ch) * 9 + k];
        return s;
    };
    auto pair_val = [&](int i, int a, int b) {   // sum (tau e2) y~_a y~_b, a <= b
        const int BA = a / 3, BB = b / 3;
        const int kind = BA * NB - BA * (BA - 1) / 2 + (BB - BA);
        return task_sum(i * (NBP + 1) + kind, (a % 3) * 3 + (b % 3));
    };
    for (int e = t; e < GK; e += TT) {
        const int i = e / K;
        int k = e % K;
        double v;
        if (k == 0) v = task_sum(i * (NBP + 1) + NBP, 0);                 // S0
        else if (k == 1) v = pair_val(i, P, P);                           // S1 = sum tau e2
        else if ((k -= 2) < P) v = pair_val(i, k, P);                     // S2
        else if ((k -= P) < P * (P + 1) / 2) {                            // S3 (upper, row-major)
            int row = 0;
            while (k >= P - row) { k -= P - row; ++row; }
            v = pair_val(i, row, row + k);
        } else v = task_sum(i * (NBP + 1) + NBP, 1);                      // S7
        out[e] = v;
    }
}

// ------------------------------------------------------------------------------------------
// q == 0, FP64-tensor-core variant (default): one warp per tile of 32 observations, no block
// barriers in the main loop.  Phase 1 (lane = observation): d, log f, tau, e2, e1-e2 for all G
// components with branch-free special functions; S0, S1, S7 accumulate per lane.  Phase 2 (warp):
// S3_i += sum_j w_ij y_j y_j' (w = tau e2) as DMMA m8n8k4: per group of 4 observations lane
// (m = lane>>2, k = lane&3) supplies a = w_{j_k} y_{j_k,m} and b = y_{j_k,m} (B's element (k, n=m)
// is the same number), so the 8x8 accumulator fragment of lane holds S3[m][2(lane&3) + {0,1}];
// S2_i[m] accumulates the same a.  Coordinates m >= p are zero padding.  DMMA runs on the FP64
// pipe (tools/bench_dmma.cu: 37 TFLOP/s alone, shared with DFMA) — the gain is issue slots: 8
// instructions per component per 32 observations instead of ~370 FFMA/LDS per observation.
#ifndef CFUST_T_MMA
#define CFUST_T_MMA 1
#endif
#ifndef CFUST_TW
#define CFUST_TW 16
#endif
constexpr int TW = CFUST_TW;   // warps per block of the q = 0 kernel
#ifndef CFUST_T_P2
#define CFUST_T_P2 2        // phase 2: 1 = w by shuffles + S2 by DADD; 2 = w rows in shared memory + S2 by one DMMA
#endif
constexpr int WSTR = 10;   // w row stride (doubles): 80-byte rows, 16-byte aligned, conflict-free 4-row reads
#ifndef CFUST_T_TAB
#define CFUST_T_TAB 0       // 1: log1p and exp of the q = 0 E-step from shared-memory tables (measured: no gain, profiles/r02k_cfg3_variants.log)
#endif
#ifndef CFUST_T_TMA
#define CFUST_T_TMA 1       // y tiles staged in shared memory by 1-D bulk copies (double-buffered)
#endif
#ifndef CFUST_T_MB
#define CFUST_T_MB 1        // blocks per SM: 16 warps in one block (profiles/r01_cfg3_mma.log)
#endif

__device__ __forceinline__ void dmma_884(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Column b of L_i^{-1} into X (stride PMAX, rows a >= b; zero elsewhere): forward substitution of
// L X = e_b, row a: X_ab = -(sum_{c=b}^{a-1} L_ac X_cb) / L_aa.
__device__ __forceinline__ void t_linv_col(const CompDev &cp, int p, int b, double *X) {
    for (int a = 0; a < PMAX; ++a) {
        double x = 0.0;
        if (a < p && b < p && a >= b) {
            if (a == b) x = cp.Linv[a];
            else {
                double r = 0.0;
                for (int c = b; c < a; ++c) r = fma(cp.L[a * PMAX + c], X[c * PMAX + b], r);
                x = -r * cp.Linv[a];
            }
        }
        X[a * PMAX + b] = x;
    }
}
__device__ __forceinline__ double t_ml_row(const CompDev &cp, int p, int a, const double *X) {
    double m = 0.0;
    for (int b = 0; b <= a && b < p; ++b) m = fma(X[a * PMAX + b], cp.mu[b], m);
    return m;
}

template <int G>
__global__ void __launch_bounds__(TW * 32, CFUST_T_MB) estep_t_mma_kernel(EArgs A, int mode) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int p = A.p, K = A.K, GK = G * K;
    CompDev *comp = reinterpret_cast<CompDev *>(smem_raw);
    double *red = reinterpret_cast<double *>(comp + G);   // [TW][GK + 1]
    for (int t = threadIdx.x; t < G * int(sizeof(CompDev) / sizeof(double)); t += blockDim.x)
        reinterpret_cast<double *>(comp)[t] = reinterpret_cast<const double *>(A.comp)[t];
    for (int t = threadIdx.x; t < TW * (GK + 1); t += blockDim.x) red[t] = 0.0;
    // L_i^{-1} (lower, row-major, stride PMAX; rows/columns >= p zero) column by column, then
    // m_i = L_i^{-1} mu_i, so that v = L^{-1}(y - mu) = L^{-1} y - m has rows independent of each
    // other (no substitution chain: 9 % faster at cfg3, profiles/r01_cfg3_mma.log).
    double *Li = red + TW * (GK + 1);                    // [G][PMAX*PMAX]
    double *mL = Li + G * PMAX * PMAX;                   // [G][PMAX]
#if CFUST_T_TMA
    // y tiles staged by the TMA engine: per warp two 32-row buffers (double buffering), each with
    // an mbarrier that the bulk copy completes; the next tile's rows land while this one computes.
    double *ybuf = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(mL + G * PMAX) + 127) & ~uintptr_t(127));   // [TW][2][32*PMAX]
    uint64_t *mbar = reinterpret_cast<uint64_t *>(ybuf + TW * 2 * 32 * PMAX);   // [TW][2]
    if (lane == 0) {
        mbar_init(mbar + 2 * wid, 1);
        mbar_init(mbar + 2 * wid + 1, 1);
        fence_proxy_async();
    }
    double *wsm_all = reinterpret_cast<double *>(mbar + 2 * TW);
#else
    double *wsm_all = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(mL + G * PMAX) + 127) & ~uintptr_t(127));
#endif
#if CFUST_T_P2 == 2
    // per warp: 32 rows of this tile's weights w_i = tau_i e2_i (i < G; entries G..7 stay zero)
    double *const wsm = wsm_all + wid * 32 * WSTR;
    for (int t = lane; t < 32 * WSTR; t += 32) wsm[t] = 0.0;
#endif
#if CFUST_T_TAB
    double2 *const ltab = reinterpret_cast<double2 *>(wsm_all + (CFUST_T_P2 == 2 ? TW * 32 * WSTR : 0));   // [128] (invc_j, log c_j)
    double *const etab = reinterpret_cast<double *>(ltab + 128);                   // [64] 2^(j/64)
    for (int t = threadIdx.x; t < 128; t += blockDim.x) {
        const double invc = (t == 0) ? 1.0 : 1.0 / (1.0 + (t + 0.5) / 128.0);
        ltab[t] = make_double2(invc, (t == 0) ? 0.0 : -log_unit(invc));
    }
    for (int t = threadIdx.x; t < 64; t += blockDim.x) etab[t] = g_EXP2J[t];
#endif
    __syncthreads();
    for (int t = threadIdx.x; t < G * PMAX; t += blockDim.x)
        t_linv_col(comp[t / PMAX], p, t % PMAX, Li + (t / PMAX) * PMAX * PMAX);
    __syncthreads();
    for (int t = threadIdx.x; t < G * PMAX; t += blockDim.x)
        mL[t] = t_ml_row(comp[t / PMAX], p, t % PMAX, Li + (t / PMAX) * PMAX * PMAX);
    __syncthreads();
    const bool nrm = A.family == 1;
    double s0[G], s1[G], s7[G], c0[G], c1[G];
#pragma unroll
    for (int i = 0; i < G; ++i) s0[i] = s1[i] = s7[i] = c0[i] = c1[i] = 0.0;
#if CFUST_T_P2 == 2
    double c20 = 0.0, c21 = 0.0;   // S2 of component cm, coordinates 2 ck, 2 ck + 1 (DMMA fragment)
#else
    double s2[G];
#pragma unroll
    for (int i = 0; i < G; ++i) s2[i] = 0.0;
#endif
    double ll = 0.0;
    const int cm = lane >> 2, ck = lane & 3;
    const int64_t n = A.n;
    const int64_t ntiles = (n + 31) / 32;
    const int64_t tstride = int64_t(gridDim.x) * TW;
#if CFUST_T_TMA
    double *const yw = ybuf + wid * 2 * 32 * PMAX;
    uint64_t *const mw = mbar + 2 * wid;
    const uint32_t tbytes = uint32_t(32 * p * sizeof(double));   // a full tile: 256 p bytes (16 | 256 p)
    // bulk copy of tile t (if it is a full one; the ragged last tile is copied by the lanes) into buffer b
    auto issue = [&](int64_t t, int b) {
        if (lane == 0 && t < ntiles && (t + 1) * 32 <= n) {
            fence_proxy_async();   // this warp's earlier generic reads of buffer b precede the async write
            mbar_expect_tx(mw + b, tbytes);
            bulk_g2s(yw + b * 32 * PMAX, A.y + t * 32 * p, tbytes, mw + b);
        }
    };
    issue(int64_t(blockIdx.x) * TW + wid, 0);
    int kk = 0;
#endif
    for (int64_t tile = int64_t(blockIdx.x) * TW + wid; tile < ntiles; tile += tstride) {
        const int64_t j = tile * 32 + lane;
        const bool valid = j < n;
        double y[PMAX];
#if CFUST_T_TMA
        const int buf = kk & 1;
        __syncwarp();   // every lane is done with buffer buf ^ 1 (the previous tile)
        issue(tile + tstride, buf ^ 1);
        double *const ys = yw + buf * 32 * PMAX;
        if ((tile + 1) * 32 <= n) {
            mbar_wait(mw + buf, (kk >> 1) & 1);
        } else {   // ragged last tile: rows past n are zero
            for (int a = 0; a < p; ++a) ys[lane * p + a] = valid ? A.y[j * p + a] : 0.0;
            __syncwarp();
        }
        ++kk;
        if (p == PMAX) {
#pragma unroll
            for (int a = 0; a < PMAX; a += 2) {
                const double2 v2 = *reinterpret_cast<const double2 *>(ys + lane * PMAX + a);
                y[a] = v2.x;
                y[a + 1] = v2.y;
            }
        } else {
#pragma unroll
            for (int a = 0; a < PMAX; ++a) y[a] = (a < p) ? ys[lane * p + a] : 0.0;
        }
#else
#if CFUST_T_P2 == 2
        __syncwarp();   // every lane is done reading the previous tile's w rows
#endif
        if (p == PMAX) {   // 64-byte rows: four 16-byte loads per lane
#pragma unroll
            for (int a = 0; a < PMAX; a += 2) {
                const double2 v2 = valid ? __ldg(reinterpret_cast<const double2 *>(A.y + j * PMAX + a)) : make_double2(0.0, 0.0);
                y[a] = v2.x;
                y[a + 1] = v2.y;
            }
        } else {
#pragma unroll
            for (int a = 0; a < PMAX; ++a) y[a] = (valid && a < p) ? __ldg(A.y + j * p + a) : 0.0;
        }
#endif
        double lf[G], dd[G], l1[G];
        double mx = -CUDART_INF;
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const CompDev &cp = comp[i];
            double d = 0.0;
            // all PMAX rows, no branch on p: rows >= p of L^{-1} and m are zero and y[a >= p] = 0, so the
            // padded rows add exactly 0 — and the scheduler interleaves rows and components (9 %)
            const double *Lr = Li + i * PMAX * PMAX, *mr = mL + i * PMAX;
#pragma unroll
            for (int a = 0; a < PMAX; ++a) {
                double t = -mr[a];
#pragma unroll
                for (int b = 0; b <= a; ++b) t = fma(Lr[a * PMAX + b], y[b], t);
                d = fma(t, t, d);
            }
            dd[i] = d;
#if CFUST_T_TAB
            l1[i] = nrm ? 0.0 : log1p_tab(d * cp.inv_nu, ltab);
#else
            l1[i] = nrm ? 0.0 : log1p_pos(d * cp.inv_nu);
#endif
            lf[i] = cp.logpi + cp.kappa - (nrm ? 0.5 * d : 0.5 * cp.m0 * l1[i]);   // normal: Gaussian component
            mx = fmax(mx, lf[i]);
        }
        double se = 0.0;
#pragma unroll
#if CFUST_T_TAB
        for (int i = 0; i < G; ++i) { lf[i] = exp_tab(lf[i] - mx, etab); se += lf[i]; }   // lf <- exp(lf - max)
#else
        for (int i = 0; i < G; ++i) { lf[i] = exp_neg(lf[i] - mx); se += lf[i]; }   // lf <- exp(lf - max)
#endif
        if (valid && mx == -CUDART_INF) atomicOr(A.status, 1);
#if CFUST_T_TAB
        if (valid) ll += mx + log_tab(se, ltab);
#else
        if (valid) ll += mx + log_unit(se);
#endif
        const double ise = div_fast(1.0, se);
        if (mode == 1) {
            if (A.tau_out && valid) {   // responsibilities and the MAP label (ties -> lowest index)
                int best = 0;
                double bv = lf[0];
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    A.tau_out[size_t(j) * G + i] = lf[i] * ise;
                    if (lf[i] > bv) { bv = lf[i]; best = i; }
                }
                A.label_out[j] = best;
            }
            continue;
        }
        double w[G];
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const CompDev &cp = comp[i];
            const double tau = valid ? lf[i] * ise : 0.0;
            const double e2 = nrm ? 1.0 : div_fast(cp.m0, cp.nu + dd[i]);
            const double e1me2 = nrm ? 0.0 : cp.psi_half_m0 - (cp.log_half_nu + l1[i]) - e2;   // log(rho/2) = log(nu/2) + log1p(d/nu)
            s0[i] += tau;
            w[i] = tau * e2;
            s1[i] += w[i];
            s7[i] = fma(tau, e1me2, s7[i]);
        }
        // phase 2: 8 groups of 4 observations
#if CFUST_T_P2 == 2
#pragma unroll
        for (int i = 0; i < G; ++i) wsm[lane * WSTR + i] = w[i];
        __syncwarp();
#endif
#pragma unroll 2
        for (int sg = 0; sg < 8; ++sg) {
#if CFUST_T_TMA
            const double yv = (cm < p) ? ys[(4 * sg + ck) * p + cm] : 0.0;
#else
            const int64_t jj = tile * 32 + 4 * sg + ck;
            const double yv = (cm < p && jj < n) ? __ldg(A.y + jj * p + cm) : 0.0;
#endif
#if CFUST_T_P2 == 2
            // S2 of every component in one DMMA: A(m = component, k) = w_{4sg+k, m}, B(k, n) = y_{4sg+k, n}
            const double *wq = wsm + (4 * sg + ck) * WSTR;
            dmma_884(c20, c21, wq[cm], yv);
#pragma unroll
            for (int i = 0; i < G; ++i) dmma_884(c0[i], c1[i], wq[i] * yv, yv);
#else
#pragma unroll
            for (int i = 0; i < G; ++i) {
                const double a = __shfl_sync(0xffffffffu, w[i], 4 * sg + ck) * yv;
                s2[i] += a;
                dmma_884(c0[i], c1[i], a, yv);
            }
#endif
        }
    }
    // ---- warp epilogue -> red[wid][*], then block sum over warps in fixed order
    double *rw = red + wid * (GK + 1);
    ll = warp_sum(ll);
    if (lane == 0) rw[GK] = ll;
    if (mode != 1) {
        const int S3o = 2 + p;   // offsets inside a component's K entries
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const double t0 = warp_sum(s0[i]), t1 = warp_sum(s1[i]), t7 = warp_sum(s7[i]);
            double *ri = rw + i * K;
            if (lane == 0) { ri[0] = t0; ri[1] = t1; ri[K - 1] = t7; }
#if CFUST_T_P2 == 2
            if (cm == i) {
                if (2 * ck < p) ri[2 + 2 * ck] = c20;
                if (2 * ck + 1 < p) ri[2 + 2 * ck + 1] = c21;
            }
#else
            double a2 = s2[i];
            a2 += __shfl_xor_sync(0xffffffffu, a2, 1);
            a2 += __shfl_xor_sync(0xffffffffu, a2, 2);
            if (ck == 0 && cm < p) ri[2 + cm] = a2;
#endif
            // S3 upper, row-major packed: entry (a, b), a <= b
            const int a = cm;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int b = 2 * ck + h;
                if (a < p && b < p && a <= b) {
                    const int off = a * p - a * (a - 1) / 2 + (b - a);
                    ri[S3o + off] = h ? c1[i] : c0[i];
                }
            }
        }
    }
    __syncthreads();
    double *out = A.partials + size_t(blockIdx.x) * (GK + 1);
    for (int e = threadIdx.x; e <= GK; e += blockDim.x) {
        if (mode == 1 && e != GK) continue;
        double v = 0.0;
        for (int wv = 0; wv < TW; ++wv) v += red[wv * (GK + 1) + e];
        out[e] = v;
    }
}

// ------------------------------------------------------------------------------------------
// Deterministic column sums of the per-block partials: block (32 x RY threads) owns 32 columns;
// thread (x, y) sums rows y, y + RY, ... in ascending order (coalesced 32-column rows), then the RY
// partial sums of a column are added in ascending y.  Fixed order -> bitwise reproducible.
constexpr int RY = 16;
__global__ void __launch_bounds__(32 * RY) reduce_kernel(const double *__restrict__ partials, int nblocks, int stride,
                                                         int col0, int ncols, double *__restrict__ out,
                                                         const int *__restrict__ flag, double *__restrict__ flag_out) {
    __shared__ double part[RY][33];
    const int x = threadIdx.x & 31, y = threadIdx.x >> 5;
    // the E-step's underflow flag (status[0] bit 0) as one more summed entry of the statistics
    // vector, so the single all-reduce also tells every rank whether some rank underflowed
    if (flag_out && blockIdx.x == 0 && threadIdx.x == 0) *flag_out = (*flag & 1) ? 1.0 : 0.0;
    const int e = blockIdx.x * 32 + x;
    double s = 0.0;
    if (e < ncols) {
#pragma unroll 4
        for (int b = y; b < nblocks; b += RY) s += partials[size_t(b) * stride + col0 + e];
    }
    part[y][x] = s;
    __syncthreads();
    if (y == 0 && e < ncols) {
        double t = 0.0;
        for (int k = 0; k < RY; ++k) t += part[k][x];
        out[e] = t;
    }
}

// q == 0 per-pair dump for parity checks: one thread per listed observation.
__global__ void dump_t_kernel(EArgs A) {
    const int g = A.g, p = A.p;
    for (int64_t jj = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; jj < A.cnt; jj += int64_t(gridDim.x) * blockDim.x) {
        const int64_t j = A.idx[jj];
        double lf[GMAX], e2[GMAX], e1me2[GMAX], mx = -CUDART_INF;
        for (int i = 0; i < g; ++i) {
            const CompDev &cp = A.comp[i];
            double v[PMAX], dd = 0.0;
            for (int a = 0; a < p; ++a) {
                double s = A.y[j * p + a] - cp.mu[a];
                for (int bb = 0; bb < a; ++bb) s -= cp.L[a * PMAX + bb] * v[bb];
                v[a] = s * cp.Linv[a];
                dd += v[a] * v[a];
            }
            const double rho = cp.nu + dd;
            if (A.family == 1) {   // Gaussian component
                lf[i] = cp.logpi + cp.kappa - 0.5 * dd;
                e2[i] = 1.0;
                e1me2[i] = 0.0;
            } else {
                lf[i] = cp.logpi + cp.kappa - 0.5 * cp.m0 * log1p(dd / cp.nu);
                e2[i] = cp.m0 / rho;
                e1me2[i] = cp.psi_half_m0 - log(0.5 * rho) - e2[i];
            }
            mx = fmax(mx, lf[i]);
        }
        double se = 0.0;
        for (int i = 0; i < g; ++i) se += exp(lf[i] - mx);
        const double lse = mx + log(se);
        double *o = A.pair_out + size_t(jj) * g * 4;
        for (int i = 0; i < g; ++i) {
            o[i * 4 + 0] = lf[i];
            o[i * 4 + 1] = exp(lf[i] - lse);
            o[i * 4 + 2] = e1me2[i];
            o[i * 4 + 3] = e2[i];
        }
    }
}

// ------------------------------------------------------------------------------------------
// Small dense helpers (single thread).
__device__ inline bool chol_dev(int n, const double *S, int lds, double *L, int ldl) {
    for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = S[i * lds + j];
            for (int k = 0; k < j; ++k) s -= L[i * ldl + k] * L[j * ldl + k];
            if (i == j) {
                if (!(s > 1e-300)) return false;
                L[i * ldl + i] = sqrt(s);
            } else {
                L[i * ldl + j] = s / L[j * ldl + j];
            }
        }
    return true;
}
__device__ inline void chol_solve_dev(int n, const double *L, int ldl, double *x) {
    for (int i = 0; i < n; ++i) {
        double s = x[i];
        for (int k = 0; k < i; ++k) s -= L[i * ldl + k] * x[k];
        x[i] = div_fast(s, L[i * ldl + i]);
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int k = i + 1; k < n; ++k) s -= L[k * ldl + i] * x[k];
        x[i] = div_fast(s, L[i * ldl + i]);
    }
}





// ------------------------------------------------------------------------------------------
// M-step (Alg. 3; reading R-M, ECM order) and the derived quantities of each
// component, one warp per component: every matrix entry is computed by one lane
// in the plain left-to-right operation order; only independent entries run in parallel.

// Cholesky of the n x n matrix A (row stride lda, n <= PMAX) into L (stride ldl; the lower triangle
// incl. the diagonal is written), left-looking column by column with row a of L in lane a's registers:
// column j takes L[j][0..j-1] from lane j by shuffles, pivot d = A_jj - sum_k L_jk^2 and
// L_aj = (A_aj - sum_k L_ak L_jk) / L_jj in ascending k.  false (in all lanes) if a pivot is <= 1e-300.
// (Round 1 staged the columns through shared memory with lane 0 computing each pivot: ~5x the latency.)
__device__ bool warp_chol(int n, const double *A, int lda, double *L, int ldl, int lane) {
    double r[PMAX];
#pragma unroll
    for (int k = 0; k < PMAX; ++k) r[k] = (lane < n && k < n) ? A[lane * lda + k] : 0.0;
    bool ok = true;
#pragma unroll
    for (int j = 0; j < PMAX; ++j) {
        if (j >= n) break;
        double v = r[j];
#pragma unroll
        for (int k = 0; k < j; ++k) v -= r[k] * __shfl_sync(0xffffffffu, r[k], j);
        const double d = __shfl_sync(0xffffffffu, v, j);
        if (!(d > 1e-300)) { ok = false; break; }
        const double ljj = sqrt_fast(d);   // rsqrt + Newton: no IEEE slow path
        if (lane == j) r[j] = ljj;
        else if (lane > j) r[j] = div_fast(v, ljj);
    }
    if (ok && lane < n) {
#pragma unroll
        for (int k = 0; k < PMAX; ++k)
            if (k <= lane) L[lane * ldl + k] = r[k];
    }
    __syncwarp();
    return ok;
}

constexpr int KMAX = 2 + PMAX + PMAX * (PMAX + 1) / 2 + QMAX + QMAX * (QMAX + 1) / 2 + PMAX * QMAX + 1;
struct MsWork {
    double Sv[KMAX];   // this component's K statistics, staged from global memory in one coalesced read
    double S3[PMAX * PMAX], S5[QMAX * QMAX], mu[PMAX], D[PMAX * QMAX], B[PMAX * QMAX], Sg[PMAX * PMAX];
    double L5[QMAX * QMAX], Lt[PMAX * PMAX];
    double md, nu;
    int ok;
};

// CFUST_MSTEP_PROF (experiment builds): clock64 stamps per warp of mstep_fused_kernel, printed at exit
#ifndef CFUST_MSTEP_PROF
#define CFUST_MSTEP_PROF 0
#endif
#if CFUST_MSTEP_PROF
__device__ long long g_mprof[2 * GMAX][24];
#define MPROF(k) do { if ((threadIdx.x & 31) == 0) g_mprof[threadIdx.x >> 5][k] = clock64(); } while (0)
#else
#define MPROF(k) do { } while (0)
#endif

__device__ double nu_update(const DevState &s, int i, double S0, double S7) {
    const double cst = S7 / S0;
    // nu: root of g(nu) = log(nu/2) - psi(nu/2) + 1 + S7/S0 on [nu_lo, nu_hi] (reading A7; g decreasing,
    // clamped when there is no sign change): safeguarded Newton from the previous nu, the bracket kept and
    // bisection taken whenever a step leaves it, to |dnu| <= 1e-13 nu (the oracle bisects to 1e-12: both
    // land within that tolerance of the root).  Called by a whole warp: lanes 0, 1, 2 evaluate g at
    // nu_hi, nu_lo and the starting point at once (one pass of the same code), then every lane runs
    // the same Newton chain (psi and psi' from one interleaved recurrence).
    const int lane = threadIdx.x & 31;
    const double lo0 = s.nu_lo, hi0 = s.nu_hi, start = fmin(fmax(s.nu[i], lo0), hi0);
    const double x0 = (lane == 0) ? hi0 : (lane == 1) ? lo0 : start;
    double ps, ps1;
    dev_psi01(0.5 * x0, ps, ps1);
    const double g0 = log_unit(0.5 * x0) - ps + 1.0 + cst;
    const double ghi = __shfl_sync(0xffffffffu, g0, 0), glo = __shfl_sync(0xffffffffu, g0, 1);
    double gv = __shfl_sync(0xffffffffu, g0, 2), psi1 = __shfl_sync(0xffffffffu, ps1, 2);
    if (ghi > 0.0) return hi0;
    if (glo < 0.0) return lo0;
    double lo = lo0, hi = hi0, nu = start;
    for (int it = 0; it < 200; ++it) {
        if (gv > 0.0) lo = nu; else hi = nu;
        const double dg = div_fast(1.0, nu) - 0.5 * psi1;
        double nn = nu - div_fast(gv, dg);
        if (!(nn > lo && nn < hi)) nn = 0.5 * (lo + hi);
        const bool done = fabs(nn - nu) <= 1e-13 * nu || hi - lo <= 1e-13 * nu;
        nu = nn;
        if (done) break;
        dev_psi01(0.5 * nu, ps, psi1);
        gv = log_unit(0.5 * nu) - ps + 1.0 + cst;
    }
    return nu;
}

__device__ int mstep_warp(const DevState &s, int i, MsWork &w, int lane, bool do_nu = true) {
    const int p = s.p, q = s.q, K = s.K;
    for (int e = lane; e < K; e += 32) w.Sv[e] = s.stats[size_t(i) * K + e];
    __syncwarp();
    MPROF(2);
    const double *S = w.Sv;
    const double S0 = S[0], S1 = S[1];
    const double *S2 = S + 2, *S3p = S2 + p, *S4 = S3p + p * (p + 1) / 2, *S5p = S4 + q;
    const double *S6 = S5p + q * (q + 1) / 2;
    const double S7 = S6[p * q];
    if (!(S0 >= 1e-10)) return -6;
    for (int e = lane; e < p * (p + 1) / 2; e += 32) {   // unpack S3 (upper, row-major)
        int a = 0, r = e;
        while (r >= p - a) { r -= p - a; ++a; }
        w.S3[a * PMAX + a + r] = S3p[e];
        w.S3[(a + r) * PMAX + a] = S3p[e];
    }
    for (int e = lane; e < q * (q + 1) / 2; e += 32) {
        int k = 0, r = e;
        while (r >= q - k) { r -= q - k; ++k; }
        w.S5[k * QMAX + k + r] = S5p[e];
        w.S5[(k + r) * QMAX + k] = S5p[e];
    }
    for (int t = lane; t < p * q; t += 32) w.D[t] = s.delta[size_t(i) * p * q + t];
    __syncwarp();
    MPROF(3);
    for (int a = lane; a < p; a += 32) {
        double v = S2[a];
        for (int k = 0; k < q; ++k) v -= w.D[a * q + k] * S4[k];
        w.mu[a] = v / S1;
    }
    __syncwarp();
    for (int t = lane; t < p * q; t += 32) {
        const int a = t / q, k = t % q;
        w.B[a * QMAX + k] = S6[a * q + k] - w.mu[a] * S4[k];
    }
    __syncwarp();
    if (q > 0) {
        if (!warp_chol(q, w.S5, QMAX, w.L5, QMAX, lane)) return -4;
        for (int a = lane; a < p; a += 32) {   // row a of B S5^{-1}
            double x[QMAX];
            for (int k = 0; k < q; ++k) x[k] = w.B[a * QMAX + k];
            chol_solve_dev(q, w.L5, QMAX, x);
            for (int k = 0; k < q; ++k) w.D[a * q + k] = x[k];
        }
        __syncwarp();
    }
    MPROF(4);
    for (int t = lane; t < p * p; t += 32) {
        const int a = t / p, b = t % p;
        double v = w.S3[a * PMAX + b] - S2[a] * w.mu[b] - w.mu[a] * S2[b] + S1 * w.mu[a] * w.mu[b];
        for (int k = 0; k < q; ++k) v -= w.B[a * QMAX + k] * w.D[b * q + k] + w.D[a * q + k] * w.B[b * QMAX + k];
        for (int k = 0; k < q; ++k)
            for (int l = 0; l < q; ++l) v += w.D[a * q + k] * w.S5[k * QMAX + l] * w.D[b * q + l];
        w.Sg[a * p + b] = v / S0;
    }
    __syncwarp();
    double sym[2] = {0.0, 0.0};
    for (int t = lane, c = 0; t < p * p; t += 32, ++c) {   // symmetrise (reads before writes)
        const int a = t / p, b = t % p;
        sym[c] = 0.5 * (w.Sg[a * p + b] + w.Sg[b * p + a]);
    }
    __syncwarp();
    for (int t = lane, c = 0; t < p * p; t += 32, ++c) {
        const int a = t / p, b = t % p;
        if (a != b) w.Sg[a * p + b] = sym[c];
    }
    __syncwarp();
    MPROF(5);
    if (!warp_chol(p, w.Sg, p, w.Lt, PMAX, lane)) {   // ridge repair
        if (lane == 0) {
            double md = 0.0;
            for (int a = 0; a < p; ++a) md += w.Sg[a * p + a];
            w.md = md / p;
        }
        __syncwarp();
        for (int a = lane; a < p; a += 32) w.Sg[a * p + a] += 1e-8 * w.md;
        __syncwarp();
        if (!warp_chol(p, w.Sg, p, w.Lt, PMAX, lane)) return -4;
    }
    MPROF(6);
    if (s.family == 1 || !do_nu) return 0;   // skew-normal / Gaussian: no nu
    const double nu = nu_update(s, i, S0, S7);   // whole warp
    if (lane == 0) w.nu = nu;
    return 0;
}

// Commit component i's M-step result (mu, Sigma, Delta in the shared MsWork; nu if solved) to the
// device parameter arrays.  Called only after every component's update succeeded, so an error
// leaves Psi^(k) intact for all components (no mix of Psi^(k) and Psi^(k+1)).
__device__ void mstep_commit(const DevState &s, int i, const MsWork &w, int lane) {
    const int p = s.p, q = s.q;
    for (int a = lane; a < p; a += 32) s.mu[size_t(i) * p + a] = w.mu[a];
    for (int t = lane; t < p * p; t += 32) s.sigma[size_t(i) * p * p + t] = w.Sg[t];
    for (int t = lane; t < p * q; t += 32) s.delta[size_t(i) * p * q + t] = w.D[t];
}

struct DvWork {
    double Sg[PMAX * PMAX], D[PMAX * QMAX], Om[PMAX * PMAX], Lc[PMAX * PMAX];
    CompDev cd;
    double lg[8];
    int ok;
};

// Derived quantities of component i, one warp, in two parts so that the fused
// M-step can run the matrix part while the nu root is still being solved:
//   derive_matrices  chol Sigma (unless supplied), Omega = Sigma + Delta Delta', its factor L, 1/L_aa,
//                    A = Delta' Omega^{-1}, Lambda = I - A Delta (symmetrised), log|Omega|, mu;
//   derive_constants the nu- and pi-dependent constants (kappa, log pi, psi(m0/2), the t_1 lgamma
//                    differences, log B(m/2, 1/2), 1/nu, log(nu/2)), then the CompDev copy-out.
// inputs_ready: w.Sg, w.D, w.cd.mu and w.Lc = chol(Sigma) already hold this component's values (the
// fused M-step supplies its own results — the same bits derive would read back and recompute).
__device__ int derive_matrices(const DevState &s, int i, DvWork &w, int lane, bool inputs_ready = false) {
    const int p = s.p, q = s.q;
    CompDev &cd = w.cd;
    if (!inputs_ready) {
        for (int t = lane; t < p * p; t += 32) w.Sg[t] = s.sigma[size_t(i) * p * p + t];
        for (int t = lane; t < p * q; t += 32) w.D[t] = s.delta[size_t(i) * p * q + t];
        for (int a = lane; a < p; a += 32) cd.mu[a] = s.mu[size_t(i) * p + a];
    }
    for (int t = lane; t < PMAX * PMAX; t += 32) { cd.L[t] = 0.0; w.Om[t] = 0.0; }
    for (int t = lane; t < QMAX * PMAX; t += 32) cd.A[t] = 0.0;
    for (int t = lane; t < QMAX * QMAX; t += 32) cd.Lam[t] = 0.0;
    __syncwarp();
    MPROF(10);
    if (!inputs_ready && !warp_chol(p, w.Sg, p, w.Lc, PMAX, lane)) return -4;   // Sigma must be PD
    MPROF(11);
    for (int t = lane; t < p * p; t += 32) {
        const int a = t / p, b = t % p;
        double v = w.Sg[a * p + b];
        for (int k = 0; k < q; ++k) v += w.D[a * q + k] * w.D[b * q + k];
        w.Om[a * PMAX + b] = v;
    }
    __syncwarp();
    if (q == 0) {   // Omega = Sigma: its factor is the one just computed (bit-identical; no second chol)
        for (int t = lane; t < PMAX * PMAX; t += 32) {
            const int a = t / PMAX, b = t % PMAX;
            cd.L[t] = (a < p && b <= a) ? w.Lc[t] : 0.0;
        }
        __syncwarp();
    } else if (!warp_chol(p, w.Om, PMAX, cd.L, PMAX, lane)) {
        return -4;
    }
    MPROF(12);
    for (int a = lane; a < PMAX; a += 32) cd.Linv[a] = (a < p) ? 1.0 / cd.L[a * PMAX + a] : 0.0;
    for (int k = lane; k < q; k += 32) {   // A = Delta' Omega^{-1}: one column of Omega^{-1} Delta per lane
        double x[PMAX];
        for (int a = 0; a < p; ++a) x[a] = w.D[a * q + k];
        chol_solve_dev(p, cd.L, PMAX, x);
        for (int a = 0; a < p; ++a) cd.A[k * PMAX + a] = x[a];
    }
    // log|Omega| = sum_a 2 log L_aa (lanes a in parallel, summed in ascending a)
    const double lv = log_unit(lane < p ? cd.L[lane * PMAX + lane] : 1.0);
    double logdet = 0.0;
    for (int a = 0; a < p; ++a) logdet += 2.0 * __shfl_sync(0xffffffffu, lv, a);
    __syncwarp();
    for (int t = lane; t < q * q; t += 32) {
        const int k = t / q, l = t % q;
        double v = 0.0;
        for (int a = 0; a < p; ++a) v += w.D[a * q + k] * cd.A[l * PMAX + a];
        cd.Lam[k * QMAX + l] = (k == l ? 1.0 : 0.0) - v;
    }
    __syncwarp();
    double sym[2] = {0.0, 0.0};
    for (int t = lane, c = 0; t < q * q; t += 32, ++c) {
        const int k = t / q, l = t % q;
        sym[c] = 0.5 * (cd.Lam[k * QMAX + l] + cd.Lam[l * QMAX + k]);
    }
    __syncwarp();
    for (int t = lane, c = 0; t < q * q; t += 32, ++c) {
        const int k = t / q, l = t % q;
        if (k != l) cd.Lam[k * QMAX + l] = sym[c];
    }
    if (lane == 0) w.lg[4] = logdet;
    __syncwarp();
    MPROF(13);
    return 0;
}

// nu = nu_i and pi = pi_i of the committed parameters; every lane on ONE code path (divergent
// branches would run one after another): lanes 0..5 lgamma at nu/2, (m0-1)/2, m0/2, (m0+1)/2,
// (m0+2)/2, (m0+3)/2; lanes 0, 1, 2 log pi_i, log(nu pi) (Gaussian family: log 2 pi), log(nu/2).
__device__ void derive_constants(const DevState &s, DvWork &w, double nu, double pii, CompDev &cd_out, int lane) {
    const int p = s.p;
    CompDev &cd = w.cd;
    const double m0 = nu + p;
    const double garg = (lane == 0) ? 0.5 * nu : 0.5 * (m0 + double(lane - 2));
    const double lgv = dev_lgamma_pos(lane < 6 ? garg : 1.0);
    MPROF(19);
    const double larg = (lane == 0) ? pii : (lane == 1) ? ((s.family == 1) ? 2.0 * CUDART_PI : nu * CUDART_PI)
                      : (lane == 2) ? 0.5 * nu : 1.0;
    const double lv = log_unit(larg);
    const double psi_m0 = dev_digamma(0.5 * m0);   // same argument in every lane: one pass
    MPROF(21);
    double G[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) G[k] = __shfl_sync(0xffffffffu, lgv, k);
    const double log_pi = __shfl_sync(0xffffffffu, lv, 0), log_nupi = __shfl_sync(0xffffffffu, lv, 1),
                 log_hnu = __shfl_sync(0xffffffffu, lv, 2);
    if (lane == 0) {
        const double logdet = w.lg[4];
        cd.nu = nu;
        cd.m0 = m0;
        cd.kappa = (s.family == 1) ? -0.5 * p * log_nupi - 0.5 * logdet   // log phi_p normaliser (log 2 pi)
                                   : (G[2] - G[0]) - 0.5 * p * log_nupi - 0.5 * logdet;
        cd.logpi = log_pi;
        cd.psi_half_m0 = psi_m0;
        cd.lgc_m0 = G[3] - G[2];     // lgamma((m0+1)/2) - lgamma(m0/2)
        cd.lgc_m0m1 = G[2] - G[1];   // lgamma(m0/2) - lgamma((m0-1)/2)
        for (int k = 0; k < 3; ++k) cd.lbt[k] = G[2 + k] + 0.5723649429247001 - G[3 + k];   // log B(m/2, 1/2), m = m0 + k
        cd.inv_nu = div_fast(1.0, nu);
        cd.log_half_nu = log_hnu;
    }
    __syncwarp();
    MPROF(14);
    double *dst = reinterpret_cast<double *>(&cd_out);
    const double *src = reinterpret_cast<const double *>(&cd);
    for (int t = lane; t < int(sizeof(CompDev) / sizeof(double)); t += 32) dst[t] = src[t];
}

__device__ int derive_warp(const DevState &s, int i, DvWork &w, CompDev &cd_out, int lane) {
    const int rc = derive_matrices(s, i, w, lane);
    if (rc != 0) return rc;
    derive_constants(s, w, s.nu[i], s.pi[i], cd_out, lane);
    return 0;
}

// M-step, one warp (block) per component; pi + derive in a second kernel after all components.
__global__ void __launch_bounds__(32) mstep_kernel(DevState s) {
    __shared__ MsWork w;
    const int i = blockIdx.x, lane = threadIdx.x;
    if (i >= s.g) return;
    const int rc = mstep_warp(s, i, w, lane);
    if (rc != 0 && lane == 0) atomicMin(s.status + 1, rc);
    if (rc != 0) return;
    __syncwarp();
    mstep_commit(s, i, w, lane);
    if (lane == 0 && s.family != 1) s.nu[i] = w.nu;
}

// pi <- S0 / n_total, floored at 1e-10, renormalised (every block recomputes the total in the same
// order), then the derived quantities of its component; skipped entirely if any M-step failed.
__global__ void __launch_bounds__(32) mstep_derive_kernel(DevState s) {
    __shared__ DvWork w;
    const int i = blockIdx.x, lane = threadIdx.x;
    if (i >= s.g || s.status[1] < 0) return;
    if (lane == 0) {
        double tot = 0.0, mine = 0.0;
        for (int c = 0; c < s.g; ++c) {
            double v = s.stats[size_t(c) * s.K] / s.n_total;
            v = (v < 1e-10) ? 1e-10 : v;
            tot += v;
            if (c == i) mine = v;
        }
        s.pi[i] = mine / tot;
    }
    __syncwarp();
    const int rc = derive_warp(s, i, w, s.comp[i], lane);
    if (rc != 0 && lane == 0) atomicMin(s.status + 1, rc);
}

// The whole M-step in one launch: one block, warp i = component i.  Phase 1 the ECM updates
// (mstep_warp); block barrier; if no component failed (status[1], which also carries earlier
// errors of the iteration), phase 2 pi and the derived quantities (derive_warp) — the same two
// steps as mstep_kernel + mstep_derive_kernel without the second launch.
union MsDvWork {
    MsWork ms;
    DvWork dv;
};
// Fit bookkeeping (DevState::fitctl, may be NULL): [0] index of the next trace slot, [1] the trace
// index at which the first error was seen (-1: none), [2] its kind (1 E-step, 2 M-step / derive).
__global__ void __launch_bounds__(64 * GMAX) mstep_fused_kernel(DevState s) {
    __shared__ MsDvWork w[GMAX];
    __shared__ double nu_new[GMAX], s0sh[GMAX];
    __shared__ int gate, slot;
    const int i = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int GK = s.g * s.K;
    MPROF(0);
    if (threadIdx.x == 0) {
        // l^(k) of the E-step that produced these statistics -> trace slot (cfust_fit, no host sync)
        int j = -1;
        if (s.fitctl) {
            j = s.fitctl[0];
            s.trace[j & (TRACE_CAP - 1)] = s.stats[GK];
            s.fitctl[0] = j + 1;
        }
        slot = j;
        // Gate: the E-step flagged an underflow on some rank (the flag travels in the statistics
        // vector through the one all-reduce, stats[GK + 1]) or non-finite data, or an earlier
        // M-step of this fit failed: Psi is left unchanged.
        const bool eflag = s.stats[GK + 1] > 0.0 || (s.status[0] & 1) || s.status[2];
        if (eflag) {
            s.status[0] |= 1;
            if (s.fitctl && s.fitctl[1] < 0) { s.fitctl[1] = j; s.fitctl[2] = 1; }
        }
        gate = eflag || s.status[1] < 0;
    }
    __syncthreads();
    MPROF(1);
    if (gate) return;
    const bool tnu = s.family != 1;   // skew-t: nu solved by warp g + i, concurrently with warp i's updates
    // This component's M-step results travel to the commit in registers (MsWork and DvWork share
    // storage, and nothing is committed before every component succeeded).
    constexpr int R2 = (PMAX * PMAX + 31) / 32, RD = (PMAX * QMAX + 31) / 32;
    double mur = 0.0, sgr[R2], dr[RD];
    if (i < s.g) {
        int rc = mstep_warp(s, i, w[i].ms, lane, false);
        if (lane == 0) s0sh[i] = w[i].ms.Sv[0];
        if (rc == 0) {
            const int p = s.p, q = s.q;
            double ltr[R2];
            if (lane < p) mur = w[i].ms.mu[lane];
#pragma unroll
            for (int c = 0; c < R2; ++c) {
                const int t = lane + 32 * c;
                sgr[c] = (t < p * p) ? w[i].ms.Sg[t] : 0.0;
                ltr[c] = w[i].ms.Lt[t];
            }
#pragma unroll
            for (int c = 0; c < RD; ++c) dr[c] = (lane + 32 * c < p * q) ? w[i].ms.D[lane + 32 * c] : 0.0;
            __syncwarp();
            DvWork &dv = w[i].dv;
            if (lane < p) dv.cd.mu[lane] = mur;
#pragma unroll
            for (int c = 0; c < R2; ++c) {
                const int t = lane + 32 * c;
                if (t < p * p) dv.Sg[t] = sgr[c];
                dv.Lc[t] = ltr[c];   // chol of exactly this Sigma (ridge repair included)
            }
#pragma unroll
            for (int c = 0; c < RD; ++c)
                if (lane + 32 * c < p * q) dv.D[lane + 32 * c] = dr[c];
            __syncwarp();
            // the derived matrices (Omega, its factor, A, Lambda, log|Omega|) overlap the nu root
            rc = derive_matrices(s, i, dv, lane, true);
        }
        if (rc != 0 && lane == 0) atomicMin(s.status + 1, rc);
        MPROF(16);
    } else if (tnu && i < 2 * s.g) {
        const int c = i - s.g;
        const double S0 = s.stats[size_t(c) * s.K], S7 = s.stats[size_t(c) * s.K + s.K - 1];
        if (S0 >= 1e-10) {   // (S0 < 1e-10: warp c reports -6)
            const double nu = nu_update(s, c, S0, S7);   // whole warp
            if (lane == 0) nu_new[c] = nu;
        }
        MPROF(7);
    }
    __syncthreads();
    MPROF(8);
    if (reinterpret_cast<volatile int *>(s.status)[1] < 0) {   // some component failed: commit nothing
        if (threadIdx.x == 0 && s.fitctl && s.fitctl[1] < 0) { s.fitctl[1] = slot; s.fitctl[2] = 2; }
        return;
    }
    if (i >= s.g) return;
    {   // commit mu, Sigma, Delta, nu of component i
        const int p = s.p, q = s.q;
        if (lane < p) s.mu[size_t(i) * p + lane] = mur;
#pragma unroll
        for (int c = 0; c < R2; ++c)
            if (lane + 32 * c < p * p) s.sigma[size_t(i) * p * p + lane + 32 * c] = sgr[c];
#pragma unroll
        for (int c = 0; c < RD; ++c)
            if (lane + 32 * c < p * q) s.delta[size_t(i) * p * q + lane + 32 * c] = dr[c];
    }
    const double nu = tnu ? nu_new[i] : s.nu[i];
    if (tnu && lane == 0) s.nu[i] = nu;
    // pi <- S0 / n_total floored at 1e-10, renormalised (lanes c < g in parallel, summed in ascending c)
    double v = (lane < s.g) ? s0sh[lane] / s.n_total : 0.0;
    v = (v < 1e-10) ? 1e-10 : v;
    double tot = 0.0;
    for (int c = 0; c < s.g; ++c) tot += __shfl_sync(0xffffffffu, v, c);
    const double pii = __shfl_sync(0xffffffffu, v, i) / tot;
    if (lane == 0) s.pi[i] = pii;
    MPROF(9);
    derive_constants(s, w[i].dv, nu, pii, s.comp[i], lane);
    MPROF(15);
#if CFUST_MSTEP_PROF
    if (lane == 0) {   // this (component) warp's stamps relative to its own start
        const long long *t = g_mprof[i];
        printf("MPROF comp %d: gate %lld stats %lld D %lld Sg %lld chol %lld dmat %lld nu %lld | bar %lld pi %lld lgam %lld cst %lld end %lld\n",
               i, t[1] - t[0], t[2] - t[0], t[4] - t[0], t[5] - t[0], t[6] - t[0], t[16] - t[0], g_mprof[s.g + i][7] - t[0],
               t[8] - t[0], t[9] - t[0], t[19] - t[0], t[21] - t[0], t[15] - t[0]);
    }
#endif
}

__global__ void __launch_bounds__(32) derive_kernel(DevState s) {
    __shared__ DvWork w;
    const int i = blockIdx.x, lane = threadIdx.x;
    if (i >= s.g) return;
    const int rc = derive_warp(s, i, w, s.comp[i], lane);
    if (rc != 0 && lane == 0) atomicMin(s.status + 1, rc);
}

// chi radius nodes: chi[(i*CHI_ROWS + k)*M + l] = sqrt(chi2_{m0+k}^{-1}(w_{l,0}) / (m0+k)), k = 0,1,2;
// row CHI_LV = log chi2_{m0}^{-1}(w_{l,0}) = log V_l (exact e1, reading R2').
// Threads take the points in ascending order of w (s.wperm): the lanes of a warp then run the same
// incomplete-gamma branch (series below a + 1, continued fraction above) for about the same number
// of terms and Newton steps, instead of both branches and the slowest lane's count.
__global__ void chi_kernel(DevState s) {
    const int M = s.M;
    const int total = s.g * CHI_ROWS * M;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int ik = t / M, i = ik / CHI_ROWS, k = ik % CHI_ROWS;
        const int l = s.wperm ? s.wperm[t % M] : t % M;
        const double w = s.W[l];   // coordinate 0 drives the chi radius
        double *out = s.chi + size_t(ik) * M + l;
        if (s.family == 1) {   // normal SOV: every radius node is 1
            *out = 1.0;
        } else if (k == CHI_LV) {   // only used (and only computed) with exact e1 / the direct estimator
            if (s.e1_exact || s.direct) *out = log(dev_chi2_quantile(w, s.comp[i].m0));
        } else {
            const double m = s.comp[i].m0 + double(k);
            *out = sqrt(dev_chi2_quantile(w, m) / m);
        }
    }
}

// wperm[rank of W[0][l]] = l (ascending, ties by l): once per context, one thread per point
__global__ void wperm_kernel(const double *__restrict__ W, int M, int *__restrict__ perm) {
    __shared__ double tile[256];
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    const double v = (l < M) ? W[l] : 0.0;
    int rank = 0;
    for (int j0 = 0; j0 < M; j0 += 256) {
        __syncthreads();
        if (j0 + int(threadIdx.x) < M && threadIdx.x < 256) tile[threadIdx.x] = W[j0 + threadIdx.x];
        __syncthreads();
        const int jn = min(256, M - j0);
        for (int j = 0; j < jn; ++j) {
            const double u = tile[j];
            rank += (u < v || (u == v && j0 + j < l)) ? 1 : 0;
        }
    }
    if (l < M) perm[rank] = l;
}

// lattice coordinates W[k][l] = |2 frac((l z_k mod M)/M + shift_k) - 1|, once per context
__global__ void lattice_kernel(DevState s, LatticeDev L) {
    const int total = s.nw * s.M;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x)
        s.W[t] = lattice_w(L, t % s.M, t / s.M);
}

__global__ void check_finite_kernel(const double *__restrict__ y, int64_t count, int *flag) {
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < count; t += int64_t(gridDim.x) * blockDim.x)
        if (!isfinite(y[t])) atomicOr(flag, 1);
}

// Diagnostic element-wise evaluation of the device special functions (cfust_eval_special).
__global__ void special_kernel(int which, const double *__restrict__ x, double *__restrict__ y, int64_t n, double aux) {
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
        const double v = x[t];
        double r;
        switch (which) {
            case 0: r = Phi(v); break;
            case 1: r = Phiinv(v); break;
            case 2: r = exp_neg(v); break;
            case 3: r = log_unit(v); break;
            case 4: r = dev_t_cdf(v, aux); break;
            case 5: r = dev_chi2_quantile(v, aux); break;
            case 6: r = dev_digamma(v); break;
            case 7: r = sqrt_fast(v); break;
            case 8: r = dev_trigamma(v); break;
            case 9: r = dev_lgamma_pos(v); break;
            case 10: r = Phi_t<true>(v); break;
            case 11: r = Phiinv_t<true>(v); break;
            case 12: r = exp_tab2(v, 0.0); break;
            default: r = CUDART_NAN;
        }
        y[t] = r;
    }
}

int launch_special(int which, const double *x, double *y, int64_t n, double aux, cudaStream_t st) {
    int64_t blocks = (n + 127) / 128;
    if (blocks < 1) blocks = 1;
    if (blocks > 4096) blocks = 4096;
    special_kernel<<<int(blocks), 128, 0, st>>>(which, x, y, n, aux);
    return int(cudaGetLastError());
}

// ------------------------------------------------------------------------------------------
// Launchers
static LatticeDev make_lattice(const DevState &s) {
    LatticeDev L;
    L.M = s.M > 0 ? s.M : 32;
    for (int k = 0; k <= QMAX; ++k) { L.z[k] = s.z[k]; L.shift[k] = s.shift[k]; }
    return L;
}

size_t comp_dev_size() { return sizeof(CompDev); }

// Fill the special-function coefficient tables of this module's constant bank.
int upload_special_constants() {
    cudaError_t e;
    if ((e = cudaMemcpyToSymbol(c_PH_P, h_PH_P, sizeof(h_PH_P))) != cudaSuccess) return int(e);
    if ((e = cudaMemcpyToSymbol(c_PH_Q, h_PH_Q, sizeof(h_PH_Q))) != cudaSuccess) return int(e);
    if ((e = cudaMemcpyToSymbol(c_NI_P, h_NI_P, sizeof(h_NI_P))) != cudaSuccess) return int(e);
    if ((e = cudaMemcpyToSymbol(c_NI_Q, h_NI_Q, sizeof(h_NI_Q))) != cudaSuccess) return int(e);
    if ((e = cudaMemcpyToSymbol(c_EXPC, h_EXPC, sizeof(h_EXPC))) != cudaSuccess) return int(e);
    if ((e = cudaMemcpyToSymbol(c_LOGC, h_LOGC, sizeof(h_LOGC))) != cudaSuccess) return int(e);
    return 0;
}

static size_t cfust_smem(const DevState &s) {
    const int GK = s.g * s.K;
    return sizeof(CompDev) * s.g + sizeof(WarpScratch) * EW + sizeof(double) * EW * (GK + 1) + sizeof(int) * GK;
}

static size_t t_smem(const DevState &s) {
    const int PE = s.p + 1, NB = (PE + 2) / 3, YS = 3 * NB, NBP = NB * (NB + 1) / 2, WS = GMAX + 1;
    const size_t tasks = size_t(s.g) * (NBP + 1) * TCH * 9;
    return sizeof(CompDev) * s.g + sizeof(double) * (size_t(TT) * (YS + 3 * WS) + 32 + tasks);
}

template <int Q, int MODE, bool DIRECT = false, int SPLIT = 1>
static int launch_cfust_q(const DevState &s, EArgs &a, cudaStream_t st, int *nb) {
    auto kern = estep_cfust_kernel<Q, MODE, DIRECT, SPLIT>;
    const size_t sm = cfust_smem(s);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    if (e != cudaSuccess) return int(e);
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, EW * 32, sm);
    if (e != cudaSuccess) return int(e);
    if (per_sm < 1) per_sm = 1;
    const int64_t work = (MODE == 2) ? a.cnt : a.n;
    int64_t blocks = int64_t(s.num_sms) * per_sm;
    const int64_t need = (work + EW / SPLIT - 1) / (EW / SPLIT);
    if (blocks > need) blocks = need;
    if (blocks < 1) blocks = 1;
    kern<<<int(blocks), EW * 32, sm, st>>>(a);
    *nb = int(blocks);
    return int(cudaGetLastError());
}

// Warps per observation for the analytic passes at small n: the largest of 1, 2, 4, 8 for which the
// n * SPLIT observation-warps fit in one wave of resident warps (num_sms x EW x the q-tuned blocks
// per SM); measured against forced values in profiles/r01_split.log.  s.split_force (env
// CFUST_SPLIT) overrides.
static int split_factor(const DevState &s) {
    if (s.direct) return 1;   // the SOV-direct pass keeps one warp per observation (T0 bits = density pass)
    if (s.split_force > 0) return s.split_force;
    const int mb = s.q == 1 ? Tune<1>::MB : s.q == 2 ? Tune<2>::MB : s.q == 3 ? Tune<3>::MB
                 : s.q == 4 ? Tune<4>::MB : s.q == 5 ? Tune<5>::MB : Tune<6>::MB;
    const int64_t cap = int64_t(s.num_sms) * EW * mb;
    int sp = 1;
    while (sp < 8 && s.n * (sp * 2) <= cap) sp *= 2;
    return sp;
}

template <int MODE, int SPLIT>
static int launch_cfust_split_q(const DevState &s, EArgs &a, cudaStream_t st, int *nb) {
    if constexpr (EW % SPLIT != 0) {   // experiment builds with small blocks (CFUST_EW < SPLIT)
        return launch_cfust_split_q<MODE, SPLIT / 2>(s, a, st, nb);
    } else {
    switch (s.q) {
        case 1: return launch_cfust_q<1, MODE, false, SPLIT>(s, a, st, nb);
        case 2: return launch_cfust_q<2, MODE, false, SPLIT>(s, a, st, nb);
        case 3: return launch_cfust_q<3, MODE, false, SPLIT>(s, a, st, nb);
        case 4: return launch_cfust_q<4, MODE, false, SPLIT>(s, a, st, nb);
        case 5: return launch_cfust_q<5, MODE, false, SPLIT>(s, a, st, nb);
        case 6: return launch_cfust_q<6, MODE, false, SPLIT>(s, a, st, nb);
        default: return int(cudaErrorInvalidValue);
    }
    }
}

template <int MODE>
static int launch_cfust_split(const DevState &s, EArgs &a, cudaStream_t st, int *nb, int sp) {
    switch (sp) {
        case 2: return launch_cfust_split_q<MODE, 2>(s, a, st, nb);
        case 4: return launch_cfust_split_q<MODE, 4>(s, a, st, nb);
        case 8: return launch_cfust_split_q<MODE, 8>(s, a, st, nb);
        default: return int(cudaErrorInvalidValue);
    }
}

template <int MODE>
static int launch_cfust_mode(const DevState &s, EArgs &a, cudaStream_t st, int *nb) {
    if constexpr (MODE != 1) {
        if (s.direct) {
            switch (s.q) {
                case 1: return launch_cfust_q<1, MODE, true>(s, a, st, nb);
                case 2: return launch_cfust_q<2, MODE, true>(s, a, st, nb);
                case 3: return launch_cfust_q<3, MODE, true>(s, a, st, nb);
                case 4: return launch_cfust_q<4, MODE, true>(s, a, st, nb);
                case 5: return launch_cfust_q<5, MODE, true>(s, a, st, nb);
                case 6: return launch_cfust_q<6, MODE, true>(s, a, st, nb);
                default: return int(cudaErrorInvalidValue);
            }
        }
    }
    if constexpr (MODE != 2) {   // statistics and density passes split alike: identical l bits
        const int sp = split_factor(s);
        if (sp > 1) return launch_cfust_split<MODE>(s, a, st, nb, sp);
    }
    switch (s.q) {
        case 1: return launch_cfust_q<1, MODE>(s, a, st, nb);
        case 2: return launch_cfust_q<2, MODE>(s, a, st, nb);
        case 3: return launch_cfust_q<3, MODE>(s, a, st, nb);
        case 4: return launch_cfust_q<4, MODE>(s, a, st, nb);
        case 5: return launch_cfust_q<5, MODE>(s, a, st, nb);
        case 6: return launch_cfust_q<6, MODE>(s, a, st, nb);
        default: return int(cudaErrorInvalidValue);
    }
}

template <int G>
static int launch_t_mma_g(const DevState &s, EArgs &a, int mode, cudaStream_t st, int *nb) {
    auto kern = estep_t_mma_kernel<G>;
    const size_t sm = sizeof(CompDev) * G + sizeof(double) * TW * (size_t(G) * s.K + 1)
                      + sizeof(double) * G * (PMAX * PMAX + PMAX)    // L^{-1}, m
                      + 128 + (CFUST_T_TMA ? sizeof(double) * TW * 2 * 32 * PMAX + sizeof(uint64_t) * TW * 2 : 0)   // y tiles, mbarriers
                      + (CFUST_T_P2 == 2 ? sizeof(double) * TW * 32 * WSTR : 0)    // w rows
                      + (CFUST_T_TAB ? sizeof(double) * (2 * 128 + 64) : 0);          // log / exp tables
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    if (e != cudaSuccess) return int(e);
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TW * 32, sm);
    if (e != cudaSuccess) return int(e);
    if (per_sm < 1) per_sm = 1;
    const int64_t ntiles = (a.n + 31) / 32;
    int64_t blocks = int64_t(s.num_sms) * per_sm;
    const int64_t need = (ntiles + TW - 1) / TW;
    if (blocks > need) blocks = need;
    if (blocks < 1) blocks = 1;
    kern<<<int(blocks), TW * 32, sm, st>>>(a, mode);
    *nb = int(blocks);
    return int(cudaGetLastError());
}

static int launch_t_mma(const DevState &s, EArgs &a, int mode, cudaStream_t st, int *nb) {
    switch (s.g) {
        case 1: return launch_t_mma_g<1>(s, a, mode, st, nb);
        case 2: return launch_t_mma_g<2>(s, a, mode, st, nb);
        case 3: return launch_t_mma_g<3>(s, a, mode, st, nb);
        case 4: return launch_t_mma_g<4>(s, a, mode, st, nb);
        case 5: return launch_t_mma_g<5>(s, a, mode, st, nb);
        case 6: return launch_t_mma_g<6>(s, a, mode, st, nb);
        case 7: return launch_t_mma_g<7>(s, a, mode, st, nb);
        case 8: return launch_t_mma_g<8>(s, a, mode, st, nb);
        default: return int(cudaErrorInvalidValue);
    }
}

template <int P>
static int launch_t_p(const DevState &s, EArgs &a, int mode, cudaStream_t st, int *nb) {
    auto kern = estep_t_kernel<P>;
    const size_t sm = t_smem(s);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    if (e != cudaSuccess) return int(e);
    const int threads = TT;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, sm);
    if (e != cudaSuccess) return int(e);
    if (per_sm < 1) per_sm = 1;
    const int64_t ntiles = (a.n + TT - 1) / TT;
    int64_t blocks = int64_t(s.num_sms) * per_sm;
    if (blocks > ntiles) blocks = ntiles;
    if (blocks < 1) blocks = 1;
    kern<<<int(blocks), threads, sm, st>>>(a, mode);
    *nb = int(blocks);
    return int(cudaGetLastError());
}

int max_partial_blocks(const DevState &s) { return s.num_sms * 32; }

int launch_estep(const DevState &s, int mode, const int64_t *idx, int64_t cnt, double *pair_out, cudaStream_t st,
                 int *nblocks_out) {
    EArgs a;
    a.y = s.y;
    a.n = s.n;
    a.p = s.p;
    a.g = s.g;
    a.K = s.K;
    a.comp = s.comp;
    a.chi = s.chi;
    a.W = s.W;
    a.M = s.M;
    a.partials = s.partials;
    a.status = s.status;
    a.idx = idx;
    a.cnt = cnt;
    a.pair_out = pair_out;
    a.e1_exact = s.e1_exact;
    a.family = s.family;
    a.direct = s.direct;
    a.tau_out = s.tau_out;
    a.label_out = s.label_out;
    *nblocks_out = 0;
    if (s.q == 0) {
        if (mode == 2) {
            int64_t blocks = (cnt + 127) / 128;
            if (blocks < 1) blocks = 1;
            dump_t_kernel<<<int(blocks > 4096 ? 4096 : blocks), 128, 0, st>>>(a);
            return int(cudaGetLastError());
        }
        if (CFUST_T_MMA) return launch_t_mma(s, a, mode, st, nblocks_out);
        switch (s.p) {
            case 1: return launch_t_p<1>(s, a, mode, st, nblocks_out);
            case 2: return launch_t_p<2>(s, a, mode, st, nblocks_out);
            case 3: return launch_t_p<3>(s, a, mode, st, nblocks_out);
            case 4: return launch_t_p<4>(s, a, mode, st, nblocks_out);
            case 5: return launch_t_p<5>(s, a, mode, st, nblocks_out);
            case 6: return launch_t_p<6>(s, a, mode, st, nblocks_out);
            case 7: return launch_t_p<7>(s, a, mode, st, nblocks_out);
            case 8: return launch_t_p<8>(s, a, mode, st, nblocks_out);
            default: return int(cudaErrorInvalidValue);
        }
    }
    switch (mode) {
        case 0: return launch_cfust_mode<0>(s, a, st, nblocks_out);
        case 1: return launch_cfust_mode<1>(s, a, st, nblocks_out);
        case 2: return launch_cfust_mode<2>(s, a, st, nblocks_out);
        default: return int(cudaErrorInvalidValue);
    }
}

// mode 1: out[0] = l, out[1] = underflow flag; otherwise out[0..GK] = statistics + l, out[GK + 1] = flag
int launch_reduce(const DevState &s, int nblocks, int mode, double *out, cudaStream_t st) {
    const int len = s.g * s.K + 1;
    if (mode == 1)   // log-likelihood only: column GK
        reduce_kernel<<<1, 32 * RY, 0, st>>>(s.partials, nblocks, len, len - 1, 1, out, s.status, out + 1);
    else
        reduce_kernel<<<(len + 31) / 32, 32 * RY, 0, st>>>(s.partials, nblocks, len, 0, len, out, s.status, out + len);
    return int(cudaGetLastError());
}

int launch_reduce_cols(const double *partials, int nblocks, int stride, int ncols, double *out, cudaStream_t st) {
    reduce_kernel<<<(ncols + 31) / 32, 32 * RY, 0, st>>>(partials, nblocks, stride, 0, ncols, out, nullptr, nullptr);
    return int(cudaGetLastError());
}

#ifndef CFUST_MSTEP_FUSED
#define CFUST_MSTEP_FUSED 1
#endif
int launch_mstep(const DevState &s, cudaStream_t st) {
#if CFUST_MSTEP_FUSED
    mstep_fused_kernel<<<1, 64 * s.g, 0, st>>>(s);
#else
    mstep_kernel<<<s.g, 32, 0, st>>>(s);
    mstep_derive_kernel<<<s.g, 32, 0, st>>>(s);
#endif
    return int(cudaGetLastError());
}
int mstep_launches() { return CFUST_MSTEP_FUSED ? 1 : 2; }

int launch_derive(const DevState &s, cudaStream_t st) {
    derive_kernel<<<s.g, 32, 0, st>>>(s);
    return int(cudaGetLastError());
}

int launch_chi(const DevState &s, cudaStream_t st) {
    if (s.M <= 0) return 0;   // no lattice: q <= 1 without exact e1
    const int total = s.g * CHI_ROWS * s.M;
    chi_kernel<<<(total + 63) / 64, 64, 0, st>>>(s);   // latency bound: spread the warps over the SMs
    return int(cudaGetLastError());
}

int launch_lattice(const DevState &s, cudaStream_t st) {
    if (s.M <= 0) return 0;
    const LatticeDev L = make_lattice(s);
    const int total = s.nw * s.M;
    lattice_kernel<<<(total + 127) / 128, 128, 0, st>>>(s, L);
    if (s.wperm) wperm_kernel<<<(s.M + 255) / 256, 256, 0, st>>>(s.W, s.M, s.wperm);
    return int(cudaGetLastError());
}

int launch_check_finite(const double *y, int64_t count, int *flag, cudaStream_t st) {
    if (count <= 0) return 0;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    check_finite_kernel<<<int(blocks), 256, 0, st>>>(y, count, flag);
    return int(cudaGetLastError());
}

}  // namespace cfust
