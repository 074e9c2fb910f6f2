// Microbenchmark: what limits the SOV loop's special functions on B200?
//  (1) throughput (warp instructions per clock per SM) of the non-DFMA instructions they issue —
//      MUFU.RCP64H (rcp.approx.ftz.f64), F2F double<->float, DSETP + FSEL selects, DADD, DMUL;
//  (2) Phi evaluations per clock per SM for variants of Phi_fast at ILP 1/2 and 16/32 warps/SM:
//      V0 production; V1 FP32 reciprocal seed + two Newton steps (no MUFU.RCP64H);
//      V2 even/odd split Horner (two half-length chains per polynomial); V3 = V1 + V2;
//      V4 V0 without the range clamp and sign select (diagnostic only);
//  (3) a dependent Phi -> Phi^{-1} -> Phi chain (the shape of one SOV point) for V0 and V3.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2005_06848_b200/csrc tools/bench_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "cfust_device.cuh"
using namespace cfust;

constexpr int ILP = 4;

__device__ __forceinline__ double rcp64(double q) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    return r;
}

// p / q with an FP32 reciprocal seed (2^-22) and two FP64 Newton steps, then the quotient correction.
__device__ __forceinline__ double div_f32seed(double p, double q) {
    float rf;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rf) : "f"(__double2float_rn(q)));
    double r = double(rf);
    double e = fma(-q, r, 1.0);
    r = fma(r, e, r);
    e = fma(-q, r, 1.0);
    r = fma(r, e, r);
    const double y = p * r;
    return fma(fma(-q, y, p), r, y);
}

// even/odd split Horner: p(x) = pe(x^2) + x po(x^2), two independent half-length chains
template <int N>
__device__ __forceinline__ double horner_eo(const double (&c)[N], double x, double x2) {
    constexpr int NE = (N + 1) / 2, NO = N / 2;
    double pe = c[2 * (NE - 1)];
#pragma unroll
    for (int k = NE - 2; k >= 0; --k) pe = fma(pe, x2, c[2 * k]);
    double po = c[2 * (NO - 1) + 1];
#pragma unroll
    for (int k = NO - 2; k >= 0; --k) po = fma(po, x2, c[2 * k + 1]);
    return fma(po, x, pe);
}

__device__ __forceinline__ double exp_neg2_eo(double xh, double xl) {
    const double t = fma(xh, 1.4426950408889634074, 6755399441055744.0);
    const int k = __double2loint(t);
    const double kd = t - 6755399441055744.0;
    const double r = fma(kd, -2.3190468138462996e-17, fma(kd, -0.69314718055994528623, xh)) + xl;
    const double p = horner_eo(c_EXPC, r, r * r);
    const double res = __hiloint2double(__double2hiint(p) + k * (1 << 20), __double2loint(p));
    return (xh < -708.0) ? 0.0 : res;
}

template <int V>
__device__ __forceinline__ double Phi_v(double x) {
    if constexpr (V == 0) {
        return Phi_fast(x);
    } else {
        const double fx = fabs(x);
        const double ax = (V == 4) ? fx : ((fx < 40.0) ? fx : 40.0);
        const double hi = ax * ax;
        const double lo = fma(ax, ax, -hi);
        double e, P, Q;
        if constexpr (V == 2 || V == 3) {
            e = exp_neg2_eo(-0.5 * hi, -0.5 * lo);
            P = horner_eo(c_PH_P, ax, hi);
            Q = horner_eo(c_PH_Q, ax, hi);
        } else {
            e = exp_neg2(-0.5 * hi, -0.5 * lo);
            P = horner_c(c_PH_P, ax);
            Q = horner_c(c_PH_Q, ax);
        }
        const double t = e * ((V == 1 || V == 3) ? div_f32seed(P, Q) : div_fast(P, Q));
        if constexpr (V == 4) return t;
        return (x < 0.0) ? t : 1.0 - t;
    }
}

template <int WHICH>
__global__ void op_kernel(double *out, int iters) {
    double x[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) x[j] = 1.25 + 1e-7 * threadIdx.x + 0.01 * j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < ILP; ++j) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if constexpr (WHICH == 0) x[j] = rcp64(x[j]);
                else if constexpr (WHICH == 1) x[j] = double(__double2float_rn(x[j]) * 1.0000001f);
                else if constexpr (WHICH == 2) x[j] = (x[j] < 1.5) ? x[j] : 1.25;
                else if constexpr (WHICH == 3) x[j] = x[j] + 1e-300;
                else if constexpr (WHICH == 4) x[j] = x[j] * 1.0000000000000002;
                else x[j] = fma(x[j], 1.0000000000000002, 1e-300);
            }
        }
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) s += x[j];
    if (s == 1234.5) out[0] = s;
}

template <int V, int IL>
__global__ void phi_kernel(double *out, int iters) {
    double x[IL], acc[IL];
#pragma unroll
    for (int j = 0; j < IL; ++j) { x[j] = -6.0 + 1e-4 * threadIdx.x + 0.37 * j; acc[j] = 0.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < IL; ++j) {
            acc[j] += Phi_v<V>(x[j]);
            x[j] += 0.0123;
            x[j] = (x[j] > 6.0) ? x[j] - 12.0 : x[j];
        }
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < IL; ++j) s += acc[j];
    if (s == 1234.5) out[0] = s;
}

// one SOV point's dependent chain: e1 = Phi(a), z = Phi^{-1}(w e1), e2 = Phi(b - c z)
template <int V, int IL>
__global__ void sov_kernel(double *out, int iters) {
    double a[IL], acc[IL];
#pragma unroll
    for (int j = 0; j < IL; ++j) { a[j] = -2.0 + 1e-4 * threadIdx.x + 0.37 * j; acc[j] = 0.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < IL; ++j) {
            const double e1 = Phi_v<V>(a[j]);
            const double w = 0.3 + 0.0001 * (it & 63);
            const double z = Phiinv(clamp_u(w * e1, UMIN, UMAX));
            const double e2 = Phi_v<V>(0.7 - 0.5 * z);
            acc[j] = fma(e1, e2, acc[j]);
            a[j] += 0.0123;
            a[j] = (a[j] > 4.0) ? a[j] - 8.0 : a[j];
        }
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < IL; ++j) s += acc[j];
    if (s == 1234.5) out[0] = s;
}

template <typename K>
float time_kernel(K kern, int blocks, int threads, double *out, int iters) {
    kern<<<blocks, threads>>>(out, 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        kern<<<blocks, threads>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double clk = 1.965e9;
    cudaMemcpyToSymbol(c_PH_P, h_PH_P, sizeof(h_PH_P));
    cudaMemcpyToSymbol(c_PH_Q, h_PH_Q, sizeof(h_PH_Q));
    cudaMemcpyToSymbol(c_EXPC, h_EXPC, sizeof(h_EXPC));
    cudaMemcpyToSymbol(c_NI_P, h_NI_P, sizeof(h_NI_P));
    cudaMemcpyToSymbol(c_NI_Q, h_NI_Q, sizeof(h_NI_Q));
    cudaMemcpyToSymbol(c_LOGC, h_LOGC, sizeof(h_LOGC));
    double *out;
    cudaMalloc(&out, 64);
    const int iters = 2048;
    const char *names[] = {"MUFU.RCP64H", "F2F f64->f32->f64 (+FMUL)", "DSETP+2xFSEL", "DADD", "DMUL", "DFMA"};
    for (int wps : {16, 32}) {
        const int blocks = sms * wps / 8;
        auto rep = [&](int w, float ms) {
            const double winst = double(iters) * ILP * 8 * (256 / 32) * blocks;   // warp-level ops
            printf("%-28s warps/SM=%2d  %8.3f ms  %.3f warp-ops/clk/SM  (%.1f lane-ops/clk/SM)\n", names[w], wps, ms,
                   winst / (ms * 1e-3) / sms / clk, 32.0 * winst / (ms * 1e-3) / sms / clk);
        };
        rep(0, time_kernel(op_kernel<0>, blocks, 256, out, iters));
        rep(1, time_kernel(op_kernel<1>, blocks, 256, out, iters));
        rep(2, time_kernel(op_kernel<2>, blocks, 256, out, iters));
        rep(3, time_kernel(op_kernel<3>, blocks, 256, out, iters));
        rep(4, time_kernel(op_kernel<4>, blocks, 256, out, iters));
        rep(5, time_kernel(op_kernel<5>, blocks, 256, out, iters));
    }
    for (int wps : {8, 16, 24, 32}) {
        const int blocks = sms * wps / 8;
        auto rp = [&](const char *nm, int il, float ms, int per) {
            const double evals = 1024.0 * il * per * 256.0 * blocks;
            printf("%-34s ilp%d warps/SM=%2d  %8.3f ms  %.3f evals/clk/SM\n", nm, il, wps, ms,
                   evals / (ms * 1e-3) / sms / clk);
        };
        rp("Phi V0 production", 1, time_kernel(phi_kernel<0, 1>, blocks, 256, out, 1024), 1);
        rp("Phi V0 production", 2, time_kernel(phi_kernel<0, 2>, blocks, 256, out, 1024), 1);
        rp("Phi V1 f32 rcp seed", 1, time_kernel(phi_kernel<1, 1>, blocks, 256, out, 1024), 1);
        rp("Phi V1 f32 rcp seed", 2, time_kernel(phi_kernel<1, 2>, blocks, 256, out, 1024), 1);
        rp("Phi V2 even/odd Horner", 1, time_kernel(phi_kernel<2, 1>, blocks, 256, out, 1024), 1);
        rp("Phi V2 even/odd Horner", 2, time_kernel(phi_kernel<2, 2>, blocks, 256, out, 1024), 1);
        rp("Phi V3 f32 seed + even/odd", 1, time_kernel(phi_kernel<3, 1>, blocks, 256, out, 1024), 1);
        rp("Phi V3 f32 seed + even/odd", 2, time_kernel(phi_kernel<3, 2>, blocks, 256, out, 1024), 1);
        rp("Phi V4 no clamp/select (diag)", 1, time_kernel(phi_kernel<4, 1>, blocks, 256, out, 1024), 1);
        rp("SOV chain V0 (evals = 3/pt)", 1, time_kernel(sov_kernel<0, 1>, blocks, 256, out, 1024), 3);
        rp("SOV chain V0 (evals = 3/pt)", 2, time_kernel(sov_kernel<0, 2>, blocks, 256, out, 1024), 3);
        rp("SOV chain V3 (evals = 3/pt)", 1, time_kernel(sov_kernel<3, 1>, blocks, 256, out, 1024), 3);
        rp("SOV chain V3 (evals = 3/pt)", 2, time_kernel(sov_kernel<3, 2>, blocks, 256, out, 1024), 3);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
