// Microbenchmark: what fraction of the B200 FP64 pipe can Horner-style code (the shape of the
// special functions in the SOV loop) reach, as a function of independent chains per thread (ILP)
// and warps per SM?  And Phi / Phi^{-1} throughput of the production device functions.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2005_06848_b200/csrc tools/bench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "cfust_device.cuh"
using namespace cfust;

__constant__ double c_H[16];

// DEG-coefficient Horner chains with constant-bank coefficients; x_j <- x_j + 1e-30 r_j keeps
// every iteration dependent on the previous one (chain length DEG per iteration).
template <int ILP>
__global__ void horner_kernel(double *out, int iters) {
    constexpr int DEG = 12;
    double x[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) x[j] = 0.25 + 1e-7 * threadIdx.x + 0.01 * j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < ILP; ++j) {
            double r = c_H[DEG - 1];
#pragma unroll
            for (int k = DEG - 2; k >= 0; --k) r = fma(r, x[j], c_H[k]);
            x[j] = fma(r, 1e-30, x[j]);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) s += x[j];
    if (s == 1234.5) out[0] = s;
}

template <int ILP, int WHICH>
__global__ void special_tp(double *out, int iters) {
    double x[ILP], acc[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) {
        x[j] = (WHICH == 0) ? -6.0 + 1e-4 * threadIdx.x + 0.37 * j : 0.001 + 1e-6 * threadIdx.x + 0.13 * j;
        acc[j] = 0.0;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < ILP; ++j) {
            if (WHICH == 0) {
                acc[j] += Phi(x[j]);
                x[j] += 0.0123;
                x[j] = (x[j] > 6.0) ? x[j] - 12.0 : x[j];
            } else {
                acc[j] += (WHICH == 1) ? Phiinv_seed(x[j]) : Phiinv_rat(x[j]);
                x[j] += 0.0123457;
                x[j] = (x[j] >= 1.0) ? x[j] - 0.9999 : x[j];
            }
        }
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) s += acc[j];
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
    int sms, clk_khz;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double clk = 1.965e9;   // max SM clock (the FP64 nominal peak's clock)
    double h[16];
    for (int k = 0; k < 16; ++k) h[k] = 1.0 / (k + 1);
    cudaMemcpyToSymbol(c_H, h, sizeof(h));
    cudaMemcpyToSymbol(c_PH_P, h_PH_P, sizeof(h_PH_P));
    cudaMemcpyToSymbol(c_PH_Q, h_PH_Q, sizeof(h_PH_Q));
    cudaMemcpyToSymbol(c_NI_P, h_NI_P, sizeof(h_NI_P));
    cudaMemcpyToSymbol(c_NI_Q, h_NI_Q, sizeof(h_NI_Q));
    cudaMemcpyToSymbol(c_EXPC, h_EXPC, sizeof(h_EXPC));
    cudaMemcpyToSymbol(c_LOGC, h_LOGC, sizeof(h_LOGC));
    double *out;
    cudaMalloc(&out, 64);
    printf("sms=%d attr_clock=%d kHz\n", sms, clk_khz);
    const int iters = 4096;
    for (int wps : {4, 8, 16, 24, 32, 48}) {   // warps per SM, 256-thread blocks
        const int blocks = sms * wps / 8;
        auto rep = [&](const char *nm, float ms, double dfma_per_thread) {
            const double total = dfma_per_thread * 256.0 * blocks;
            const double per_clk_sm = total / (ms * 1e-3) / sms / clk;
            printf("horner %-5s warps/SM=%2d  %.3f ms  DFMA/clk/SM=%.1f  (%.0f%% of 64)\n", nm, wps, ms, per_clk_sm,
                   100.0 * per_clk_sm / 64.0);
        };
        rep("ilp1", time_kernel(horner_kernel<1>, blocks, 256, out, iters), 12.0 * iters * 1);
        rep("ilp2", time_kernel(horner_kernel<2>, blocks, 256, out, iters), 12.0 * iters * 2);
        rep("ilp3", time_kernel(horner_kernel<3>, blocks, 256, out, iters), 12.0 * iters * 3);
        rep("ilp4", time_kernel(horner_kernel<4>, blocks, 256, out, iters), 12.0 * iters * 4);
    }
    const int it2 = 1024;
    for (int wps : {8, 16, 32}) {
        const int blocks = sms * wps / 8;
        auto rep = [&](const char *nm, float ms, int ilp) {
            const double evals = double(it2) * ilp * 256.0 * blocks;
            printf("%-12s warps/SM=%2d  %.3f ms  %.3e evals/s  %.2f evals/clk/SM\n", nm, wps, ms, evals / (ms * 1e-3),
                   evals / (ms * 1e-3) / sms / clk);
        };
        rep("Phi ilp1", time_kernel(special_tp<1, 0>, blocks, 256, out, it2), 1);
        rep("Phi ilp2", time_kernel(special_tp<2, 0>, blocks, 256, out, it2), 2);
        rep("Phiinv ilp1", time_kernel(special_tp<1, 1>, blocks, 256, out, it2), 1);
        rep("Phiinv ilp2", time_kernel(special_tp<2, 1>, blocks, 256, out, it2), 2);
        rep("Phiinv_rat 1", time_kernel(special_tp<1, 2>, blocks, 256, out, it2), 1);
        rep("Phiinv_rat 2", time_kernel(special_tp<2, 2>, blocks, 256, out, it2), 2);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
