/*
 * cfust_fit.c — the C ABI without Python: fit a g-component CFUST mixture (arXiv 2005.06848,
 * Eq. (2); EM of Algs. 2-4) on one GPU and print the log-likelihood trace and the MAP labels' sizes.
 *
 *   gcc -O2 examples/cfust_fit.c -Iinclude -Lpaper_2005_06848_b200 -lcfust \
 *       -Wl,-rpath,$PWD/paper_2005_06848_b200 -o cfust_fit
 *   ./cfust_fit problem.bin 20
 *
 * problem.bin (little-endian, written by examples/write_problem.py):
 *   int32 n, p, q, g, M, s; then double y[n][p], pi[g], mu[g][p], sigma[g][p][p], delta[g][p][q],
 *   nu[g]; then (M > 0) uint32 z[s], double shift[s] (the lattice's s coordinates, include/cfust.h).
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "cfust.h"

static void *read_exact(FILE *f, size_t bytes) {
    void *p = malloc(bytes ? bytes : 1);
    if (!p || fread(p, 1, bytes, f) != bytes) { fprintf(stderr, "short read\n"); exit(2); }
    return p;
}

int main(int argc, char **argv) {
    if (argc < 2) { fprintf(stderr, "usage: %s problem.bin [max_iter]\n", argv[0]); return 2; }
    const int max_iter = argc > 2 ? atoi(argv[2]) : 10;
    FILE *f = fopen(argv[1], "rb");
    if (!f) { perror(argv[1]); return 2; }
    int32_t hdr[6];
    if (fread(hdr, sizeof(int32_t), 6, f) != 6) { fprintf(stderr, "bad header\n"); return 2; }
    const int n = hdr[0], p = hdr[1], q = hdr[2], g = hdr[3], M = hdr[4], nz = hdr[5];
    double *y = read_exact(f, sizeof(double) * (size_t)n * p);
    cfust_params init;
    init.pi = read_exact(f, sizeof(double) * g);
    init.mu = read_exact(f, sizeof(double) * g * p);
    init.sigma = read_exact(f, sizeof(double) * g * p * p);
    init.delta = read_exact(f, sizeof(double) * g * p * q);
    init.nu = read_exact(f, sizeof(double) * g);
    cfust_opts opts = {0};
    uint32_t *z = NULL;
    double *shift = NULL;
    if (M > 0) {
        z = read_exact(f, sizeof(uint32_t) * nz);
        shift = read_exact(f, sizeof(double) * nz);
        opts.lattice_m = M;
        opts.lattice_z = z;
        opts.lattice_shift = shift;
    }
    fclose(f);
    opts.device = -1;
    opts.world = 1;

    cfust_ctx *ctx = NULL;
    int rc = cfust_em_init(&ctx, y, n, p, g, q, &init, &opts);
    if (rc != CFUST_OK) { fprintf(stderr, "cfust_em_init: %d\n", rc); return 1; }
    double *trace = malloc(sizeof(double) * (max_iter + 1));
    cfust_result res = {0};
    res.loglik_trace = trace;
    res.trace_cap = max_iter + 1;
    rc = cfust_fit(ctx, max_iter, 0.0, &res);
    if (rc != CFUST_OK) { fprintf(stderr, "cfust_fit: %d (%s)\n", rc, cfust_last_error(ctx)); return 1; }
    for (int k = 0; k <= res.n_iter; ++k) printf("loglik[%d] = %.10f\n", k, trace[k]);
    int32_t *labels = malloc(sizeof(int32_t) * (n ? n : 1));
    double ll = 0.0;
    rc = cfust_predict(ctx, labels, NULL, &ll);
    if (rc != CFUST_OK) { fprintf(stderr, "cfust_predict: %d\n", rc); return 1; }
    int *counts = calloc(g, sizeof(int));
    for (int j = 0; j < n; ++j) counts[labels[j]]++;
    printf("iterations %d, wall %.3f s, final loglik %.10f\ncluster sizes:", res.n_iter, res.wall_time_s, ll);
    for (int i = 0; i < g; ++i) printf(" %d", counts[i]);
    printf("\n");
    cfust_destroy(ctx);
    return 0;
}
