// Microbenchmark: FP64 tensor-core MMA (mma.sync m8n8k4 f64 -> SASS DMMA) throughput on B200,
// alone and interleaved with independent DFMA chains (does DMMA use a pipe separate from DFMA?).
// Decides the design of the q = 0 E-step's statistics contraction.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int CH, int NF>
__global__ void mix_kernel(double *out, int iters) {
    double c[CH > 0 ? CH : 1][2];
    double a = 1.0 + 1e-9 * threadIdx.x, b = 0.999;
    double x[NF > 0 ? NF : 1];
#pragma unroll
    for (int k = 0; k < CH; ++k) c[k][0] = c[k][1] = 0.0;
#pragma unroll
    for (int k = 0; k < NF; ++k) x[k] = threadIdx.x * 1e-7 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < CH; ++k) dmma(c[k], a, b);
#pragma unroll
        for (int k = 0; k < NF; ++k) x[k] = fma(x[k], 0.9999999, 1e-9);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < CH; ++k) s += c[k][0] + c[k][1];
#pragma unroll
    for (int k = 0; k < NF; ++k) s += x[k];
    if (s == 1234.5) out[0] = s;
}

template <int CH, int NF>
void run(int sms, double *out) {
    const int blocks = sms * 4, threads = 256, iters = 4096;
    mix_kernel<CH, NF><<<blocks, threads>>>(out, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        mix_kernel<CH, NF><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double warps = blocks * threads / 32.0;
    const double mma_flops = 2.0 * 8 * 8 * 4 * CH * double(iters) * warps;
    const double fma_flops = 2.0 * NF * double(iters) * blocks * threads;
    printf("DMMA chains=%d DFMA chains=%d: %.3f ms  DMMA %.2f TFLOP/s  DFMA %.2f TFLOP/s  total %.2f\n", CH, NF, best,
           mma_flops / best / 1e9, fma_flops / best / 1e9, (mma_flops + fma_flops) / best / 1e9);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 64);
    run<1, 0>(sms, out);
    run<2, 0>(sms, out);
    run<4, 0>(sms, out);
    run<8, 0>(sms, out);
    run<0, 8>(sms, out);
    run<4, 8>(sms, out);
    run<2, 8>(sms, out);
    run<4, 16>(sms, out);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
