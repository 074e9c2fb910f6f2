// Experiment: the SOV point loop with the special-function coefficients held in REGISTERS
// (loaded once per thread) instead of read from the constant bank at every evaluation
// (LDC/LDCU per coefficient pair).  Same arithmetic as Phi_fast / Phiinv_seed.
#include <cstdio>
#include <cuda_runtime.h>
#include "cfust_device.cuh"
using namespace cfust;

struct Coef {
    double P[11], Q[12], E[14];
};

template <int N>
__device__ __forceinline__ double horner_r(const double (&c)[N], double x) {
    double r = c[N - 1];
#pragma unroll
    for (int k = N - 2; k >= 0; --k) r = fma(r, x, c[k]);
    return r;
}

__device__ __forceinline__ double exp_r(double x, const Coef &C) {
    const double t = fma(x, 1.4426950408889634074, 6755399441055744.0);
    const int k = __double2loint(t);
    const double kd = t - 6755399441055744.0;
    const double r = fma(kd, -2.3190468138462996e-17, fma(kd, -0.69314718055994528623, x));
    const double p = horner_r(C.E, r);
    const double res = __hiloint2double(__double2hiint(p) + k * (1 << 20), __double2loint(p));
    return (x < -708.0) ? 0.0 : res;
}

__device__ __forceinline__ double Phi_r(double x, const Coef &C) {
    const double fx = fabs(x);
    const double ax = (fx < 40.0) ? fx : 40.0;
    const double hi = ax * ax;
    const double lo = fma(ax, ax, -hi);
    const double e = exp_r(-0.5 * hi, C) * (1.0 - 0.5 * lo);
    const double t = e * div_fast(horner_r(C.P, ax), horner_r(C.Q, ax));
    return (x < 0.0) ? t : 1.0 - t;
}

__device__ __forceinline__ double Phiinv_r(double u, const Coef &C) {
    const double uc = 1.0 - u;
    const double t = (u < uc) ? u : uc;
    const int hx = __double2hiint(t);
    const float m = __int_as_float(0x3f800000 | ((hx & 0x000fffff) << 3));
    const float e2t = float((hx >> 20) - 1022);
    float w = -0.6931471806f * (e2t + lg2_ftz(m));
    w = fmaxf(w, 0.0f);
    const float v = (w > 0.0f) ? w * rsqrt_ftz(w) : 0.0f;
    const double ax = fmin(double(w * seed_U32(v)), 37.5);
    const double hi = ax * ax;
    const double lo = fma(ax, ax, -hi);
    const double ep = exp_r(0.5 * hi, C) * (1.0 + 0.5 * lo);
    const double R = div_fast(horner_r(C.P, ax), horner_r(C.Q, ax));
    const double r = 2.5066282746310002 * fma(t, ep, -R);
    const double xx = fma(r, fma(r, fma(r, (2.0 * hi + 1.0) * (1.0 / 6.0), -0.5 * ax), 1.0), -ax);
    return (u < 0.5) ? xx : -xx;
}

template <int R, int MINB, bool REG>
__global__ void __launch_bounds__(256, MINB) sov_bench(const double* __restrict__ chi, const double* __restrict__ W,
                                                      int M, int npairs, double* out) {
    Coef C;
    if (REG) {
#pragma unroll
        for (int k = 0; k < 11; ++k) C.P[k] = c_PH_P[k];
#pragma unroll
        for (int k = 0; k < 12; ++k) C.Q[k] = c_PH_Q[k];
#pragma unroll
        for (int k = 0; k < 14; ++k) C.E[k] = c_EXPC[k];
    }
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    double tot = 0.0;
    for (int pr = warp; pr < npairs; pr += nw) {
        double binv[R], Cn[R * (R - 1) / 2];
#pragma unroll
        for (int k = 0; k < R; ++k) binv[k] = 0.3 - 0.2 * k + 1e-3 * (pr & 7);
#pragma unroll
        for (int k = 0; k < R * (R - 1) / 2; ++k) Cn[k] = 0.1 * (k % 3) - 0.05;
        double acc = 0.0;
        for (int l = lane; l < M; l += 32) {
            const double s = __ldg(chi + l);
            double e = REG ? Phi_r(s * binv[0], C) : Phi(s * binv[0]);
            double f = e;
            double z[R - 1];
#pragma unroll
            for (int k = 1; k < R; ++k) {
                const double w = __ldg(W + k * M + l);
                double u = w * e;
                u = (u < UMIN) ? UMIN : u;
                u = (u > UMAX) ? UMAX : u;
                z[k - 1] = REG ? Phiinv_r(u, C) : Phiinv(u);
                double a = s * binv[k];
#pragma unroll
                for (int t = 0; t < k; ++t) a -= Cn[(k * (k - 1)) / 2 + t] * z[t];
                e = REG ? Phi_r(a, C) : Phi(a);
                f *= e;
            }
            acc += f;
        }
        tot += warp_sum(acc);
    }
    if (lane == 0) out[warp] = tot;
}

__global__ void fill(double* chi, double* W, int M) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < M) { chi[t] = 0.5 + 1.0 * ((t * 7919) % M) / M; }
    if (t < 6 * M) W[t] = ((t * 104729) % 1000003) / 1000003.0 * 0.999 + 0.0005;
}

template <int R, int MINB, bool REG>
void run(const char* name, double* chi, double* W, int M, int npairs, double* out, int sms) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sov_bench<R, MINB, REG>, 256, 0);
    int blocks = sms * per_sm;
    cudaFuncAttributes at; cudaFuncGetAttributes(&at, sov_bench<R, MINB, REG>);
    sov_bench<R, MINB, REG><<<blocks, 256>>>(chi, W, M, npairs, out);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    sov_bench<R, MINB, REG><<<blocks, 256>>>(chi, W, M, npairs, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double evals = double(npairs) * M * (2 * R - 1);
    printf("%s R=%d reg=%d regs=%d warps/SM=%d  %.3f ms  %.3e evals/s\n", name, R, int(REG), at.numRegs, per_sm * 8, ms,
           evals / (ms * 1e-3));
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int M = 2048, npairs = 148 * 64 * 8;
    double *chi, *W, *out;
    cudaMalloc(&chi, M * 8); cudaMalloc(&W, 6 * M * 8); cudaMalloc(&out, 1 << 24);
    fill<<<(6 * M + 255) / 256, 256>>>(chi, W, M);
    cudaMemcpyToSymbol(c_PH_P, h_PH_P, sizeof(h_PH_P));
    cudaMemcpyToSymbol(c_PH_Q, h_PH_Q, sizeof(h_PH_Q));
    cudaMemcpyToSymbol(c_NI_P, h_NI_P, sizeof(h_NI_P));
    cudaMemcpyToSymbol(c_NI_Q, h_NI_Q, sizeof(h_NI_Q));
    cudaMemcpyToSymbol(c_EXPC, h_EXPC, sizeof(h_EXPC));
    cudaMemcpyToSymbol(c_LOGC, h_LOGC, sizeof(h_LOGC));
    run<4, 1, false>("minb1", chi, W, M, npairs, out, sms);
    run<4, 1, true>("minb1", chi, W, M, npairs, out, sms);
    run<4, 2, false>("minb2", chi, W, M, npairs, out, sms);
    run<4, 2, true>("minb2", chi, W, M, npairs, out, sms);
    run<3, 2, false>("minb2", chi, W, M, npairs, out, sms);
    run<3, 2, true>("minb2", chi, W, M, npairs, out, sms);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
