// Microbenchmark: the SOV point loop alone (T_R lattice rule with the production Phi/Phiinv),
// at several occupancies, to see what the hot loop can reach without the per-pair setup.
#include <cstdio>
#include <cuda_runtime.h>
#include "cfust_device.cuh"
using namespace cfust;

template <int R, int MINB>
__global__ void __launch_bounds__(256, MINB) sov_bench(const double* __restrict__ chi, const double* __restrict__ W,
                                                      int M, int npairs, double* out) {
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
            double e = Phi(s * binv[0]);
            double f = e;
            double z[R - 1];
#pragma unroll
            for (int k = 1; k < R; ++k) {
                const double w = __ldg(W + k * M + l);
                double u = w * e;
            u = (u < UMIN) ? UMIN : u;
            u = (u > UMAX) ? UMAX : u;
            z[k - 1] = Phiinv(u);
                double a = s * binv[k];
#pragma unroll
                for (int t = 0; t < k; ++t) a -= Cn[(k * (k - 1)) / 2 + t] * z[t];
                e = Phi(a);
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

template <int R, int MINB>
void run(const char* name, double* chi, double* W, int M, int npairs, double* out, int sms) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sov_bench<R, MINB>, 256, 0);
    int blocks = sms * per_sm;
    cudaFuncAttributes at; cudaFuncGetAttributes(&at, sov_bench<R, MINB>);
    sov_bench<R, MINB><<<blocks, 256>>>(chi, W, M, npairs, out);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    sov_bench<R, MINB><<<blocks, 256>>>(chi, W, M, npairs, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double evals = double(npairs) * M * (2 * R - 1);
    printf("%s R=%d regs=%d warps/SM=%d  %.3f ms  %.3e evals/s  %.1f ns/eval/SM\n", name, R, at.numRegs, per_sm * 8, ms,
           evals / (ms * 1e-3), ms * 1e6 * sms / evals);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int M = 2048, npairs = 148 * 64 * 8;
    double *chi, *W, *out;
    cudaMalloc(&chi, M * 8); cudaMalloc(&W, 6 * M * 8); cudaMalloc(&out, 1 << 24);
    fill<<<(6 * M + 255) / 256, 256>>>(chi, W, M);
    // constants
    extern int upload_special_constants_tool();
    upload_special_constants_tool();
    run<4, 1>("minb1", chi, W, M, npairs, out, sms);
    run<4, 2>("minb2", chi, W, M, npairs, out, sms);
    run<4, 3>("minb3", chi, W, M, npairs, out, sms);
    run<4, 4>("minb4", chi, W, M, npairs, out, sms);
    run<2, 4>("minb4", chi, W, M, npairs, out, sms);
    run<6, 4>("minb4", chi, W, M, npairs, out, sms);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

int upload_special_constants_tool() {
    cudaMemcpyToSymbol(c_PH_P, h_PH_P, sizeof(h_PH_P));
    cudaMemcpyToSymbol(c_PH_Q, h_PH_Q, sizeof(h_PH_Q));
    cudaMemcpyToSymbol(c_NI_P, h_NI_P, sizeof(h_NI_P));
    cudaMemcpyToSymbol(c_NI_Q, h_NI_Q, sizeof(h_NI_Q));
    cudaMemcpyToSymbol(c_EXPC, h_EXPC, sizeof(h_EXPC));
    cudaMemcpyToSymbol(c_LOGC, h_LOGC, sizeof(h_LOGC));
    return 0;
}
