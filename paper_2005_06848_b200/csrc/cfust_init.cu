// cfust_init.cu — kernels of Alg. 1, the parallel multi-start initialisation (
// SURVEY.md §8(f) NEXT-1), under readings I1-I4 of DESIGN.md §3:
//   random_labels_kernel     I1  counter-based random partitions (splitmix64 of (seed, stream, j))
//   mind_kernel / argmax_*   I2  farthest-point seeding and empty-cluster re-seeding
//   assign_kernel            I2  Lloyd assignment (nearest centre, ties -> lowest index)
//   part_sums_kernel         I2/I3 per-component sums over a hard partition, deterministic
//                                (contiguous row chunks per block, fixed in-block order; the
//                                blocks are combined by reduce_kernel in ascending order)
//   centers_kernel           I2  centre = member mean (empty clusters flagged for re-seeding)
//   partition_params_kernel  I3  Psi^(0) from the partition moments, written into Psi on device
// Distances are accumulated d = fma(t, t, d) over ascending coordinates (as the oracle does), so
// seeding and assignment decisions are bit-identical to it given identical centres.
#include "cfust_device.cuh"
#include "cfust_internal.h"

namespace cfust {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void random_labels_kernel(int32_t *__restrict__ lab, int64_t n, int64_t j0, int g, uint64_t seed,
                                     int64_t stream) {
    const uint64_t key = splitmix64(splitmix64(seed) ^ uint64_t(stream));
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t h = splitmix64(key ^ uint64_t(j0 + j));
        lab[j] = int32_t((h >> 32) % uint64_t(g));
    }
}

__device__ __forceinline__ double sqdist(const double *__restrict__ a, const double *__restrict__ b, int p) {
    double d = 0.0;
    for (int k = 0; k < p; ++k) {
        const double t = a[k] - b[k];
        d = fma(t, t, d);
    }
    return d;
}

// mind[j] = |y_j - c|^2 (init) or min(mind[j], |y_j - c|^2)
__global__ void mind_kernel(const double *__restrict__ y, int64_t n, int p, const double *__restrict__ c,
                            double *__restrict__ mind, int init) {
    double cc[PMAX];
    for (int k = 0; k < p; ++k) cc[k] = c[k];
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
        const double d = sqdist(y + j * p, cc, p);
        mind[j] = init ? d : fmin(mind[j], d);
    }
}

// argmax over j of v[j] with ties -> lowest j; partial per block (value, global index)
__global__ void argmax_partial_kernel(const double *__restrict__ v, int64_t n, int64_t j0, double *__restrict__ pval,
                                      int64_t *__restrict__ pidx) {
    __shared__ double sv[256];
    __shared__ int64_t si[256];
    double bv = -1.0;
    int64_t bi = INT64_MAX;
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
        const double x = v[j];
        if (x > bv) { bv = x; bi = j0 + j; }   // ascending j per thread: strict > keeps the lowest
    }
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            const double ov = sv[threadIdx.x + s];
            const int64_t oi = si[threadIdx.x + s];
            if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
                sv[threadIdx.x] = ov;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        pval[blockIdx.x] = sv[0];
        pidx[blockIdx.x] = si[0];
    }
}

__global__ void argmax_final_kernel(const double *__restrict__ pval, const int64_t *__restrict__ pidx, int nb,
                                    double *__restrict__ out /* [2]: value, index as double */) {
    if (threadIdx.x != 0) return;
    double bv = -1.0;
    int64_t bi = INT64_MAX;
    for (int b = 0; b < nb; ++b)
        if (pval[b] > bv || (pval[b] == bv && pidx[b] < bi)) { bv = pval[b]; bi = pidx[b]; }
    out[0] = bv;
    out[1] = double(bi);
}

// Lloyd assignment: nearest centre (ties -> lowest index); per-block count of changed labels
__global__ void assign_kernel(const double *__restrict__ y, int64_t n, int p, int g, const double *__restrict__ cen,
                              int32_t *__restrict__ lab, double *__restrict__ mind, double *__restrict__ pchanged) {
    __shared__ double sc[GMAX * PMAX];
    __shared__ int cnt[256];
    for (int t = threadIdx.x; t < g * p; t += blockDim.x) sc[t] = cen[t];
    __syncthreads();
    int changed = 0;
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
        const double *yj = y + j * p;
        int bi = 0;
        double bd = sqdist(yj, sc, p);
        for (int i = 1; i < g; ++i) {
            const double d = sqdist(yj, sc + i * p, p);
            if (d < bd) { bd = d; bi = i; }
        }
        if (lab[j] != bi) { lab[j] = bi; ++changed; }
        mind[j] = bd;
    }
    cnt[threadIdx.x] = changed;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) cnt[threadIdx.x] += cnt[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) pchanged[blockIdx.x] = double(cnt[0]);
}

// Per-component sums over a hard partition.  pass 1: [count, sum y (p)] per component;
// pass 2 (t = y - ybar_i): [sum t t' (upper p(p+1)/2, row-major), sum t^3 (p)] per component.
// Block b owns rows [b chunk, (b+1) chunk), staged TILE rows at a time in shared memory; each
// statistics entry is owned by one thread and accumulated in ascending row order.
constexpr int PS_TILE = 128;
constexpr int PS_THREADS = 256;

__global__ void __launch_bounds__(PS_THREADS) part_sums_kernel(const double *__restrict__ y, int64_t n, int p, int g,
                                                               const int32_t *__restrict__ lab,
                                                               const double *__restrict__ ybar, int pass,
                                                               int64_t chunk, double *__restrict__ partials) {
    __shared__ double ty[PS_TILE * PMAX];
    __shared__ int32_t tl[PS_TILE];
    __shared__ double sb[GMAX * PMAX];
    const int per = (pass == 1) ? 1 + p : p * (p + 1) / 2 + p;
    const int E = g * per;
    if (pass == 2)
        for (int t = threadIdx.x; t < g * p; t += blockDim.x) sb[t] = ybar[t];
    constexpr int EPT = (GMAX * (PMAX * (PMAX + 1) / 2 + PMAX) + PS_THREADS - 1) / PS_THREADS;   // entries per thread
    double acc[EPT];
    int ent_i[EPT], ent_a[EPT], ent_b[EPT];   // component, coordinates (b = -1: linear / count)
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        acc[k] = 0.0;
        const int e = threadIdx.x + k * PS_THREADS;
        ent_i[k] = -1;
        if (e < E) {
            const int i = e / per;
            int r = e % per;
            ent_i[k] = i;
            if (pass == 1) {
                ent_a[k] = r - 1;   // -1: count
                ent_b[k] = -1;
            } else if (r < p * (p + 1) / 2) {
                int row = 0;
                while (r >= p - row) { r -= p - row; ++row; }
                ent_a[k] = row;
                ent_b[k] = row + r;
            } else {
                ent_a[k] = r - p * (p + 1) / 2;
                ent_b[k] = -2;      // cube
            }
        }
    }
    const int64_t r0 = int64_t(blockIdx.x) * chunk;
    const int64_t r1 = (r0 + chunk < n) ? r0 + chunk : n;
    for (int64_t t0 = r0; t0 < r1; t0 += PS_TILE) {
        const int rows = int((r1 - t0 < PS_TILE) ? r1 - t0 : PS_TILE);
        __syncthreads();
        for (int t = threadIdx.x; t < rows * p; t += blockDim.x) ty[t] = y[t0 * p + t];
        for (int t = threadIdx.x; t < rows; t += blockDim.x) tl[t] = lab[t0 + t];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            const int i = ent_i[k];
            if (i < 0) continue;
            const int a = ent_a[k], b = ent_b[k];
            double s = acc[k];
            for (int r = 0; r < rows; ++r) {
                if (tl[r] != i) continue;
                const double *yr = ty + r * p;
                if (pass == 1) {
                    s += (a < 0) ? 1.0 : yr[a];
                } else if (b >= 0) {
                    s += (yr[a] - sb[i * p + a]) * (yr[b] - sb[i * p + b]);
                } else {
                    const double t = yr[a] - sb[i * p + a];
                    s += t * t * t;
                }
            }
            acc[k] = s;
        }
    }
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        const int e = threadIdx.x + k * PS_THREADS;
        if (e < E) partials[size_t(blockIdx.x) * E + e] = acc[k];
    }
}

// centre / mean of each component from pass-1 sums: out[i][k] = sum_ik / count_i (count 0:
// out unchanged, empty[i] = 1)
__global__ void centers_kernel(const double *__restrict__ sums1, int p, int g, double *__restrict__ out,
                               int *__restrict__ empty) {
    const int i = threadIdx.x;
    if (i >= g) return;
    const double *s = sums1 + i * (1 + p);
    const double c = s[0];
    empty[i] = (c > 0.0) ? 0 : 1;
    if (c > 0.0)
        for (int k = 0; k < p; ++k) out[i * p + k] = s[1 + k] / c;
}

// Psi^(0) from the partition moments (reading I3), written into Psi on the device.
// valid[0] = 0 if a component has < p+1 members or a non-PD covariance.
__global__ void partition_params_kernel(DevState s, const double *__restrict__ sums1, const double *__restrict__ sums2,
                                        const double *__restrict__ ybar, int *__restrict__ valid) {
    const int i = threadIdx.x;
    const int p = s.p, q = s.q, g = s.g;
    if (i >= g) return;
    const double ni = sums1[i * (1 + p)];
    if (!(ni >= double(p + 1))) { atomicAnd(valid, 0); return; }
    const int per = p * (p + 1) / 2 + p;
    const double *m2 = sums2 + i * per;
    double S[PMAX * PMAX];
    int o = 0;
    for (int a = 0; a < p; ++a)
        for (int b = a; b < p; ++b) { S[a * p + b] = S[b * p + a] = m2[o] / ni; ++o; }
    // Cholesky test of S (pivot > 1e-300)
    double L[PMAX * PMAX];
    for (int a = 0; a < p; ++a)
        for (int b = 0; b <= a; ++b) {
            double v = S[a * p + b];
            for (int k = 0; k < b; ++k) v -= L[a * PMAX + k] * L[b * PMAX + k];
            if (a == b) {
                if (!(v > 1e-300)) { atomicAnd(valid, 0); return; }
                L[a * PMAX + a] = sqrt(v);
            } else {
                L[a * PMAX + b] = v / L[b * PMAX + b];
            }
        }
    double *D = s.delta + size_t(i) * p * q;
    for (int t = 0; t < p * q; ++t) D[t] = 0.0;
    for (int k = 0; k < p && k < q; ++k) D[k * q + k] = (m2[o + k] < 0.0 ? -0.5 : 0.5) * sqrt(S[k * p + k]);
    for (int a = 0; a < p; ++a) {
        double t = 0.0;
        for (int k = 0; k < q; ++k) t += D[a * q + k];
        s.mu[size_t(i) * p + a] = ybar[i * p + a] - sqrt(2.0 / CUDART_PI) * t;
    }
    for (int t = 0; t < p * p; ++t) s.sigma[size_t(i) * p * p + t] = S[t];
    s.nu[i] = 10.0;
    s.pi[i] = ni / s.n_total;
}

// ------------------------------------------------------------------------------------------
// Launchers
static int grid_for(int64_t n, int threads, int cap) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return int(b);
}

int launch_random_labels(int32_t *lab, int64_t n, int64_t j0, int g, uint64_t seed, int64_t stream, cudaStream_t st) {
    if (n <= 0) return 0;
    random_labels_kernel<<<grid_for(n, 256, 4096), 256, 0, st>>>(lab, n, j0, g, seed, stream);
    return int(cudaGetLastError());
}

int launch_mind(const double *y, int64_t n, int p, const double *c, double *mind, int init, cudaStream_t st) {
    if (n <= 0) return 0;
    mind_kernel<<<grid_for(n, 256, 4096), 256, 0, st>>>(y, n, p, c, mind, init);
    return int(cudaGetLastError());
}

// (value, global index) of the local argmax into out[2] (device); scratch >= 2 * 1024 doubles
int launch_argmax(const double *v, int64_t n, int64_t j0, double *scratch, double *out, cudaStream_t st) {
    const int nb = grid_for(n, 256, 1024);
    double *pval = scratch;
    int64_t *pidx = reinterpret_cast<int64_t *>(scratch + 1024);
    argmax_partial_kernel<<<nb, 256, 0, st>>>(v, n > 0 ? n : 0, j0, pval, pidx);
    argmax_final_kernel<<<1, 32, 0, st>>>(pval, pidx, nb, out);
    return int(cudaGetLastError());
}

// changed-label count -> out[0] (device, via the partials reduction)
int launch_assign(const double *y, int64_t n, int p, int g, const double *cen, int32_t *lab, double *mind,
                  double *partials, int *nb_out, cudaStream_t st) {
    const int nb = grid_for(n, 256, 2048);
    assign_kernel<<<nb, 256, 0, st>>>(y, n, p, g, cen, lab, mind, partials);
    *nb_out = nb;
    return int(cudaGetLastError());
}

int part_sums_width(int p, int g, int pass) { return g * ((pass == 1) ? 1 + p : p * (p + 1) / 2 + p); }

int launch_part_sums(const double *y, int64_t n, int p, int g, const int32_t *lab, const double *ybar, int pass,
                     int max_blocks, double *partials, int *nb_out, cudaStream_t st) {
    int64_t nb = (n + 4 * PS_TILE - 1) / (4 * PS_TILE);
    if (nb > max_blocks) nb = max_blocks;
    if (nb < 1) nb = 1;
    const int64_t chunk = (n + nb - 1) / nb;
    part_sums_kernel<<<int(nb), PS_THREADS, 0, st>>>(y, n, p, g, lab, ybar, pass, chunk > 0 ? chunk : 1, partials);
    *nb_out = int(nb);
    return int(cudaGetLastError());
}

int launch_centers(const double *sums1, int p, int g, double *out, int *empty, cudaStream_t st) {
    centers_kernel<<<1, 32, 0, st>>>(sums1, p, g, out, empty);
    return int(cudaGetLastError());
}

int launch_partition_params(const DevState &s, const double *sums1, const double *sums2, const double *ybar, int *valid,
                            cudaStream_t st) {
    partition_params_kernel<<<1, 32, 0, st>>>(s, sums1, sums2, ybar, valid);
    return int(cudaGetLastError());
}

}  // namespace cfust
