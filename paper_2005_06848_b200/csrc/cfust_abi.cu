// cfust_abi.cu — host side of libcfust.so: context, validation, NCCL, and the C ABI
// declared in include/cfust.h.  Every step of the hot path runs in cfust_kernels.cu; this
// file only allocates, launches, and moves the O(g K) statistics vector.
#include "cfust.h"
#include "cfust_device.cuh"
#include "cfust_internal.h"

#include <nccl.h>
#ifndef CFUST_NVTX
#define CFUST_NVTX 1
#endif
#if CFUST_NVTX
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost a pointer test unless a tool attaches
#endif

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

using namespace cfust;

struct cfust_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    DevState s{};
    double *y_owned = nullptr;
    double *d_ll = nullptr;        // loglik-only result
    double *h_pin = nullptr;       // pinned: [0] loglik, [1..] stats staging
    int *h_status = nullptr;       // pinned [4]
    ncclComm_t comm = nullptr;
    bool comm_failed = false;      // an NCCL error or timeout aborted the communicator: every call fails
    int world = 1, rank = 0;
    bool have_stats = false;
    bool timing = false;
    cudaEvent_t ev[5] = {};
    double ms[4] = {0, 0, 0, 0};
    int64_t counts[4] = {0, 0, 0, 0};
    int64_t launches = 0;
    int nblocks_last = 0;
    int64_t j0 = 0;                // global index of the first local observation
    // CUDA graphs of one EM iteration (captured on first use; no timing events inside):
    //   [0] cfust_iterate order  E-step -> reduce -> all-reduce -> M-step -> chi nodes
    //   [1] cfust_fit order      M-step -> chi nodes -> E-step -> reduce -> all-reduce
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    int64_t glaunches[2] = {0, 0}; // kernels of ours per graph launch (NCCL's not counted)
    int *h_fitctl = nullptr;       // pinned [4]: fit bookkeeping staging (DevState::fitctl)
    double *h_trace = nullptr;     // pinned [TRACE_CAP]
    // Alg. 1 workspace (allocated on first use)
    int32_t *d_labels = nullptr;   // [m_cap][n]
    int m_cap = 0;
    double *d_init = nullptr;      // mind[n] | cent[g p] | ybar[g p] | sums1 | sums2 | argmax scratch
    int *d_iflag = nullptr;        // [GMAX + 1]: empty flags, valid
    double *h_ipin = nullptr;      // pinned staging for Alg. 1 scalars
    double *d_tau = nullptr;       // cfust_predict outputs
    int32_t *d_lab = nullptr;
    std::string err;
};

namespace {

// NVTX ranges (SURVEY §5 tracing): one per C-ABI call and per phase of an iteration, so an nsys /
// ncu --nvtx timeline attributes kernels to E-step, reduction, all-reduce and M-step.
struct Nvtx {
    explicit Nvtx(const char *name) {
#if CFUST_NVTX
        nvtxRangePushA(name);
#else
        (void)name;
#endif
    }
    ~Nvtx() {
#if CFUST_NVTX
        nvtxRangePop();
#endif
    }
    Nvtx(const Nvtx &) = delete;
    Nvtx &operator=(const Nvtx &) = delete;
};

int fail(cfust_ctx *c, int code, const std::string &msg) {
    if (c) c->err = msg;
    return code;
}

// A local CUDA failure on a multi-rank context: abort the communicator so that the peers' next
// collective fails (their waits poll ncclCommGetAsyncError) instead of blocking on this rank.
int fail_local(cfust_ctx *c, int code, const std::string &msg) {
    if (c && c->comm && c->world > 1) {
        ncclCommAbort(c->comm);
        c->comm = nullptr;
        c->comm_failed = true;
    }
    return fail(c, code, msg);
}

#define CU(call)                                                                                        \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess) return fail_local(ctx, CFUST_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define CUI(call)                                                                                       \
    do {                                                                                                \
        int e_ = (call);                                                                                \
        if (e_ != 0) return fail_local(ctx, CFUST_ECUDA, std::string(#call) + ": " + cudaGetErrorString(cudaError_t(e_))); \
    } while (0)

#define NC(call)                                                                                        \
    do {                                                                                                \
        ncclResult_t r_ = (call);                                                                       \
        if (r_ != ncclSuccess) return fail(ctx, CFUST_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)

int k_stats(int p, int q) { return 3 + p + p * (p + 1) / 2 + q + q * (q + 1) / 2 + p * q; }

// Host-side validation of Psi.
int validate_params(cfust_ctx *ctx, int p, int q, int g, const cfust_params *P) {
    if (!P || !P->pi || !P->mu || !P->sigma || !P->nu || (q > 0 && !P->delta))
        return fail(ctx, CFUST_EINVAL, "NULL parameter array");
    double tot = 0.0;
    for (int i = 0; i < g; ++i) {
        if (!(P->pi[i] > 0.0)) return fail(ctx, CFUST_EMIXPROP, "pi_i <= 0");
        tot += P->pi[i];
        if (!(P->nu[i] > 0.0) || !std::isfinite(P->nu[i])) return fail(ctx, CFUST_EINVAL, "nu_i must be > 0");
    }
    if (!(std::fabs(tot - 1.0) <= 1e-12)) return fail(ctx, CFUST_EMIXPROP, "|sum pi - 1| > 1e-12");
    for (int t = 0; t < g * p; ++t)
        if (!std::isfinite(P->mu[t])) return fail(ctx, CFUST_EINVAL, "mu not finite");
    for (int i = 0; i < g; ++i)
        for (int a = 0; a < p; ++a)
            for (int b = 0; b < p; ++b) {
                const double x = P->sigma[(size_t(i) * p + a) * p + b], y = P->sigma[(size_t(i) * p + b) * p + a];
                if (!std::isfinite(x)) return fail(ctx, CFUST_EINVAL, "Sigma not finite");
                if (std::fabs(x - y) > 1e-12 * (std::fabs(x) + std::fabs(y) + 1e-300))
                    return fail(ctx, CFUST_EDIM, "Sigma not symmetric");
            }
    for (int t = 0; t < g * p * q; ++t)
        if (!std::isfinite(P->delta[t])) return fail(ctx, CFUST_EINVAL, "Delta not finite");
    return CFUST_OK;
}

int upload_params(cfust_ctx *ctx, const cfust_params *P) {
    DevState &s = ctx->s;
    const int p = s.p, q = s.q, g = s.g;
    CU(cudaMemcpyAsync(s.pi, P->pi, sizeof(double) * g, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyAsync(s.mu, P->mu, sizeof(double) * g * p, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyAsync(s.sigma, P->sigma, sizeof(double) * g * p * p, cudaMemcpyHostToDevice, ctx->stream));
    if (q > 0) CU(cudaMemcpyAsync(s.delta, P->delta, sizeof(double) * g * p * q, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyAsync(s.nu, P->nu, sizeof(double) * g, cudaMemcpyHostToDevice, ctx->stream));
    return CFUST_OK;
}

// status word -> error code (after a stream sync).  uflag: the all-reduced E-step underflow flag
// (statistics vector entry g*K+1, or d_ll[1] of a density pass) when the caller fetched one; < 0:
// use this rank's status[0] (set on every rank by the M-step gate from the same global flag).
int check_status(cfust_ctx *ctx, double uflag = -1.0) {
    const int *st = ctx->h_status;
    if (st[1] < 0) {
        const int code = st[1];
        return fail(ctx, code, code == CFUST_ENOTPD ? "matrix not positive definite (Cholesky pivot <= 1e-300)"
                               : code == CFUST_EEMPTY ? "empty component: S0_i < 1e-10"
                                                      : "M-step/derive error");
    }
    if ((uflag >= 0.0) ? (uflag > 0.0) : (st[0] & 1))
        return fail(ctx, CFUST_EUNDERFLOW, "all component densities underflow at some observation");
    if (st[2]) return fail(ctx, CFUST_EINVAL, "y has non-finite entries");
    return CFUST_OK;
}

// Wait for the context stream.  With a communicator the wait polls (cudaStreamQuery) and checks
// ncclCommGetAsyncError, and optionally a deadline, so that a failed or vanished peer turns into
// CFUST_ENCCL on this rank (communicator aborted) instead of a hang — fail fast, SURVEY §5.
int wait_stream(cfust_ctx *ctx) {
    if (ctx->comm_failed) return fail(ctx, CFUST_ENCCL, "communicator aborted by an earlier NCCL failure");
    if (!ctx->comm) {
        CU(cudaStreamSynchronize(ctx->stream));
        return CFUST_OK;
    }
    // read per wait (settable at any time); with world > 1 a finite default, so a peer that died
    // before a collective cannot block this rank forever
    const char *to = std::getenv("CFUST_NCCL_TIMEOUT_S");
    const double timeout_s = to ? std::atof(to) : (ctx->world > 1 ? 1800.0 : 0.0);
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t q = cudaStreamQuery(ctx->stream);
        if (q == cudaSuccess) return CFUST_OK;
        if (q != cudaErrorNotReady) return fail(ctx, CFUST_ECUDA, cudaGetErrorString(q));
        ncclResult_t ae = ncclSuccess;
        const ncclResult_t r = ncclCommGetAsyncError(ctx->comm, &ae);
        std::string why;
        if (r != ncclSuccess || ae != ncclSuccess)
            why = std::string("NCCL async error: ") + ncclGetErrorString(r != ncclSuccess ? r : ae);
        else if (timeout_s > 0.0 &&
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s)
            why = "collective wait exceeded CFUST_NCCL_TIMEOUT_S";
        if (!why.empty()) {
            ncclCommAbort(ctx->comm);
            ctx->comm = nullptr;
            ctx->comm_failed = true;
            return fail(ctx, CFUST_ENCCL, why);
        }
        std::this_thread::yield();
    }
}

int fetch_status_and_sync(cfust_ctx *ctx, const double *uflag_host = nullptr) {
    CU(cudaMemcpyAsync(ctx->h_status, ctx->s.status, sizeof(int) * 4, cudaMemcpyDeviceToHost, ctx->stream));
    const int rc = wait_stream(ctx);
    if (rc) return rc;
    return check_status(ctx, uflag_host ? *uflag_host : -1.0);
}

void rec(cfust_ctx *ctx, int k) {
    if (ctx->timing) cudaEventRecord(ctx->ev[k], ctx->stream);
}

void acc_phase(cfust_ctx *ctx, int a, int b, int slot) {
    if (!ctx->timing) return;
    float t = 0.f;
    if (cudaEventElapsedTime(&t, ctx->ev[a], ctx->ev[b]) == cudaSuccess) {
        ctx->ms[slot] += t;
        ctx->counts[slot] += 1;
    }
}

int reset_status(cfust_ctx *ctx) {
    if (ctx->comm_failed) return fail(ctx, CFUST_ENCCL, "communicator aborted by an earlier NCCL failure");
    CU(cudaMemsetAsync(ctx->s.status, 0, sizeof(int) * 4, ctx->stream));
    return CFUST_OK;
}

// Context creation (world > 1): agree on the status word over ranks with ONE collective (max of
// [underflow, -code, non-finite]) so that every rank returns the same code.  Not used per
// iteration: there the E-step's underflow flag rides in the statistics all-reduce and the M-step's
// codes are identical on all ranks (same inputs, same kernel).
int global_status(cfust_ctx *ctx) {
    if (!ctx->comm) return CFUST_OK;
    CU(cudaMemcpyAsync(ctx->h_status, ctx->s.status, sizeof(int) * 4, cudaMemcpyDeviceToHost, ctx->stream));
    int rc = wait_stream(ctx);
    if (rc) return rc;
    int *h = ctx->h_status;
    h[1] = -h[1];
    CU(cudaMemcpyAsync(ctx->s.status, h, sizeof(int) * 4, cudaMemcpyHostToDevice, ctx->stream));
    NC(ncclAllReduce(ctx->s.status, ctx->s.status, 3, ncclInt32, ncclMax, ctx->comm, ctx->stream));
    CU(cudaMemcpyAsync(h, ctx->s.status, sizeof(int) * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if ((rc = wait_stream(ctx))) return rc;
    h[1] = -h[1];
    CU(cudaMemcpyAsync(ctx->s.status, h, sizeof(int) * 4, cudaMemcpyHostToDevice, ctx->stream));
    return CFUST_OK;
}

// E-step (mode 0) or loglik (mode 1) up to the global reduction; no host sync.  The reduced vector
// (statistics + l + underflow flag, or l + flag) is all-reduced by exactly ONE collective.
int enqueue_estep(cfust_ctx *ctx, int mode) {
    DevState &s = ctx->s;
    int nb = 0;
    rec(ctx, 0);
    {
        Nvtx r(mode == 1 ? "cfust:loglik-kernel" : "cfust:estep-kernel");
        CUI(launch_estep(s, mode, nullptr, 0, nullptr, ctx->stream, &nb));
    }
    ctx->launches += 1;
    rec(ctx, 1);
    {
        Nvtx r("cfust:reduce");
        CUI(launch_reduce(s, nb, mode, mode == 1 ? ctx->d_ll : s.stats, ctx->stream));
    }
    ctx->launches += 1;
    rec(ctx, 2);
    ctx->nblocks_last = nb;
    if (ctx->comm) {
        Nvtx r("cfust:allreduce");
        const size_t len = (mode == 1) ? 2 : size_t(s.g) * s.K + 2;
        NC(ncclAllReduce(mode == 1 ? ctx->d_ll : s.stats, mode == 1 ? ctx->d_ll : s.stats, len, ncclDouble, ncclSum,
                         ctx->comm, ctx->stream));
    }
    rec(ctx, 3);
    return CFUST_OK;
}

int enqueue_mstep(cfust_ctx *ctx) {
    Nvtx r("cfust:mstep");
    CUI(launch_mstep(ctx->s, ctx->stream));
    CUI(launch_chi(ctx->s, ctx->stream));
    ctx->launches += mstep_launches() + ((ctx->s.M > 0) ? 1 : 0);   // M-step (+ pi, derive), chi nodes
    rec(ctx, 4);
    return CFUST_OK;
}

bool use_graphs(const cfust_ctx *ctx) {
    static const bool off = std::getenv("CFUST_NO_GRAPH") != nullptr;
    return !ctx->timing && !off;   // per-phase timing events stay on the eager path
}

void drop_graphs(cfust_ctx *ctx) {
    for (auto &g : ctx->gexec)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
}

// One EM iteration as a CUDA graph (which = 0: E then M, cfust_iterate; 1: M then E, cfust_fit),
// captured on first use from the same enqueue functions as the eager path; eager when timing.
int enqueue_iteration(cfust_ctx *ctx, int which) {
    auto body = [&]() {
        int r = (which == 0) ? enqueue_estep(ctx, 0) : enqueue_mstep(ctx);
        if (r == CFUST_OK) r = (which == 0) ? enqueue_mstep(ctx) : enqueue_estep(ctx, 0);
        return r;
    };
    if (!use_graphs(ctx)) return body();
    if (!ctx->gexec[which]) {
        const int64_t l0 = ctx->launches;
        CU(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        int rc = body();
        cudaGraph_t g = nullptr;
        const cudaError_t ee = cudaStreamEndCapture(ctx->stream, &g);
        if (rc == CFUST_OK && ee != cudaSuccess) rc = fail_local(ctx, CFUST_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ee));
        if (rc == CFUST_OK && cudaGraphInstantiate(&ctx->gexec[which], g, 0) != cudaSuccess)
            rc = fail_local(ctx, CFUST_ECUDA, "cudaGraphInstantiate failed");
        if (g) cudaGraphDestroy(g);
        ctx->glaunches[which] = ctx->launches - l0;
        ctx->launches = l0;
        if (rc) { ctx->gexec[which] = nullptr; return rc; }
    }
    CU(cudaGraphLaunch(ctx->gexec[which], ctx->stream));
    ctx->launches += ctx->glaunches[which];
    return CFUST_OK;
}

}  // namespace

extern "C" {

int cfust_k_stats(int32_t p, int32_t q) { return k_stats(p, q); }

int cfust_nccl_unique_id(void *out) {
    if (!out) return CFUST_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return CFUST_ENCCL;
    std::memcpy(out, &id, sizeof(id));
    return CFUST_OK;
}

const char *cfust_last_error(const cfust_ctx *ctx) { return ctx ? ctx->err.c_str() : "NULL context"; }

void *cfust_stream(cfust_ctx *ctx) { return ctx ? (void *)ctx->stream : nullptr; }

int64_t cfust_launch_count(cfust_ctx *ctx) { return ctx ? ctx->launches : 0; }

void cfust_destroy(cfust_ctx *ctx) {
    if (!ctx) return;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    drop_graphs(ctx);
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    DevState &s = ctx->s;
    cudaFree(s.trace);
    cudaFree(s.fitctl);
    cudaFreeHost(ctx->h_fitctl);
    cudaFreeHost(ctx->h_trace);
    cudaFree(ctx->y_owned);
    cudaFree(s.pi);
    cudaFree(s.mu);
    cudaFree(s.sigma);
    cudaFree(s.delta);
    cudaFree(s.nu);
    cudaFree(s.comp);
    cudaFree(s.chi);
    cudaFree(s.W);
    cudaFree(s.wperm);
    cudaFree(s.partials);
    cudaFree(s.stats);
    cudaFree(s.status);
    cudaFree(ctx->d_ll);
    cudaFree(ctx->d_labels);
    cudaFree(ctx->d_init);
    cudaFree(ctx->d_iflag);
    cudaFreeHost(ctx->h_ipin);
    cudaFree(ctx->d_tau);
    cudaFree(ctx->d_lab);
    cudaFreeHost(ctx->h_pin);
    cudaFreeHost(ctx->h_status);
    for (auto &e : ctx->ev)
        if (e) cudaEventDestroy(e);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int cfust_em_init(cfust_ctx **out, const double *y, int64_t n, int32_t p, int32_t g, int32_t q,
                  const cfust_params *init, const cfust_opts *opts) {
    Nvtx nvtx_range("cfust_em_init");
    if (!out) return CFUST_EINVAL;
    *out = nullptr;
    cfust_ctx *ctx = new cfust_ctx();
    int rc = CFUST_OK;
    do {
        if (!opts) { rc = fail(ctx, CFUST_EINVAL, "opts is NULL"); break; }
        if (p < 1 || p > PMAX || q < 0 || q > QMAX || g < 1 || g > GMAX || n < 0) {
            rc = fail(ctx, CFUST_EDIM, "need 1<=p<=8, 0<=q<=6, 1<=g<=8, n>=0");
            break;
        }
        if (n > 0 && !y) { rc = fail(ctx, CFUST_EINVAL, "y is NULL"); break; }
        if (opts->family < 0 || opts->family > 1) { rc = fail(ctx, CFUST_EINVAL, "family must be 0 (skew-t) or 1 (skew-normal)"); break; }
        if (opts->estimator < 0 || opts->estimator > 1) { rc = fail(ctx, CFUST_EINVAL, "estimator must be 0 (analytic) or 1 (SOV-direct)"); break; }
        const bool direct = opts->estimator == 1 && q >= 1;   // SOV-direct truncated moments (reading D1)
        const bool use_e1 = (opts->e1_exact != 0 || direct) && q >= 1 && opts->family == 0;   // q = 0: A5 exact; no W for skew-normal
        const bool need_lat = q >= 2 || use_e1 || direct;
        const int M = need_lat ? opts->lattice_m : 0;
        const int nz = direct ? q + 1 : (q > 1 ? q : 1);      // lattice coordinates used
        if (need_lat) {
            if (M < 1024 || M > 65536 || (M & (M - 1)) != 0) {
                rc = fail(ctx, CFUST_EINVAL, "lattice_m must be a power of two in [1024, 65536]");
                break;
            }
            if (!opts->lattice_z || !opts->lattice_shift) { rc = fail(ctx, CFUST_EINVAL, "lattice z/shift NULL"); break; }
            for (int k = 0; k < nz; ++k) {
                if (opts->lattice_z[k] == 0 || opts->lattice_z[k] >= uint32_t(M)) { rc = fail(ctx, CFUST_EINVAL, "bad lattice z"); break; }
                if (!(opts->lattice_shift[k] > 0.0 && opts->lattice_shift[k] < 1.0)) { rc = fail(ctx, CFUST_EINVAL, "lattice shift must be in (0,1)"); break; }
            }
            if (rc != CFUST_OK) break;
        }
        rc = validate_params(ctx, p, q, g, init);
        if (rc != CFUST_OK) break;
        ctx->world = opts->world > 1 ? opts->world : 1;
        ctx->rank = opts->rank;
        ctx->j0 = opts->global_offset > 0 ? opts->global_offset : 0;
        ctx->timing = opts->timing != 0;
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) { rc = fail(ctx, CFUST_ECUDA, "no CUDA device"); break; }
        ctx->device = opts->device >= 0 ? opts->device : 0;
        if (opts->device < 0) cudaGetDevice(&ctx->device);
        if (cudaSetDevice(ctx->device) != cudaSuccess) { rc = fail(ctx, CFUST_ECUDA, "cudaSetDevice failed"); break; }
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, ctx->device) != cudaSuccess) { rc = fail(ctx, CFUST_ECUDA, "cudaGetDeviceProperties"); break; }
        if (prop.major < 10) { rc = fail(ctx, CFUST_ECUDA, "libcfust is built for sm_100a (B200)"); break; }
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) { rc = fail(ctx, CFUST_ECUDA, "stream"); break; }
        if (upload_special_constants() != 0) { rc = fail(ctx, CFUST_ECUDA, "constant upload failed"); break; }
        for (auto &e : ctx->ev)
            if (cudaEventCreate(&e) != cudaSuccess) { rc = fail(ctx, CFUST_ECUDA, "event"); break; }
        if (rc != CFUST_OK) break;
        DevState &s = ctx->s;
        s.p = p; s.q = q; s.g = g; s.K = k_stats(p, q);
        s.n = n;
        s.n_total = opts->n_total > 0 ? double(opts->n_total) : double(n);
        s.nu_lo = (opts->nu_lo > 0.0) ? opts->nu_lo : 0.1;
        s.nu_hi = (opts->nu_hi > 0.0) ? opts->nu_hi : 1000.0;
        s.M = M;
        for (int k = 0; k < 8; ++k) { s.z[k] = 1; s.shift[k] = 0.5; }
        for (int k = 0; k < nz && M > 0; ++k) { s.z[k] = opts->lattice_z[k]; s.shift[k] = opts->lattice_shift[k]; }
        s.e1_exact = use_e1 ? 1 : 0;
        s.family = opts->family;
        s.direct = direct ? 1 : 0;
        s.nw = nz;
        {   // CFUST_SPLIT=1|2|4|8: force the warps-per-observation of the small-n statistics pass (tests)
            const char *sp = std::getenv("CFUST_SPLIT");
            const int v = sp ? std::atoi(sp) : 0;
            s.split_force = (v == 1 || v == 2 || v == 4 || v == 8) ? v : 0;
        }
        s.num_sms = prop.multiProcessorCount;
        const int GK1 = g * s.K + 1;
        auto alloc = [&](void **ptr, size_t bytes) { return cudaMalloc(ptr, bytes < 8 ? 8 : bytes) == cudaSuccess; };
        bool ok = alloc((void **)&s.pi, sizeof(double) * g) && alloc((void **)&s.mu, sizeof(double) * g * p) &&
                  alloc((void **)&s.sigma, sizeof(double) * g * p * p) &&
                  alloc((void **)&s.delta, sizeof(double) * g * p * (q > 0 ? q : 1)) &&
                  alloc((void **)&s.nu, sizeof(double) * g) && alloc((void **)&s.comp, comp_dev_size() * g) &&
                  alloc((void **)&s.chi, sizeof(double) * g * CHI_ROWS * (M > 0 ? M : 1)) &&
                  alloc((void **)&s.W, sizeof(double) * nz * (M > 0 ? M : 1)) &&
                  alloc((void **)&s.wperm, sizeof(int) * (M > 0 ? M : 1)) &&
                  alloc((void **)&s.partials, sizeof(double) * size_t(max_partial_blocks(s)) * GK1) &&
                  alloc((void **)&s.stats, sizeof(double) * (GK1 + 1)) && alloc((void **)&s.status, sizeof(int) * 4) &&
                  alloc((void **)&ctx->d_ll, sizeof(double) * 2) &&
                  alloc((void **)&s.trace, sizeof(double) * TRACE_CAP) && alloc((void **)&s.fitctl, sizeof(int) * 4);
        if (!ok) { rc = fail(ctx, CFUST_ECUDA, "cudaMalloc failed"); break; }
        if (cudaMemsetAsync(s.stats, 0, sizeof(double) * (GK1 + 1), ctx->stream) != cudaSuccess ||
            cudaMemsetAsync(s.fitctl, 0, sizeof(int) * 4, ctx->stream) != cudaSuccess) {
            rc = fail(ctx, CFUST_ECUDA, "cudaMemset failed");
            break;
        }
        if (cudaMallocHost((void **)&ctx->h_pin, sizeof(double) * (GK1 + 2)) != cudaSuccess ||
            cudaMallocHost((void **)&ctx->h_status, sizeof(int) * 4) != cudaSuccess ||
            cudaMallocHost((void **)&ctx->h_fitctl, sizeof(int) * 4) != cudaSuccess ||
            cudaMallocHost((void **)&ctx->h_trace, sizeof(double) * TRACE_CAP) != cudaSuccess) {
            rc = fail(ctx, CFUST_ECUDA, "cudaMallocHost failed");
            break;
        }
        if (opts->y_on_device) {
            s.y = y;
        } else {
            if (cudaMalloc((void **)&ctx->y_owned, sizeof(double) * (n > 0 ? n * p : 1)) != cudaSuccess) {
                rc = fail(ctx, CFUST_ECUDA, "cudaMalloc y failed");
                break;
            }
            if (n > 0 && cudaMemcpyAsync(ctx->y_owned, y, sizeof(double) * n * p, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess) {
                rc = fail(ctx, CFUST_ECUDA, "copy y failed");
                break;
            }
            s.y = ctx->y_owned;
        }
        rc = reset_status(ctx);
        if (rc != CFUST_OK) break;
        rc = upload_params(ctx, init);
        if (rc != CFUST_OK) break;
        if (launch_check_finite(s.y, n * p, s.status + 2, ctx->stream) != 0 || launch_lattice(s, ctx->stream) != 0 ||
            launch_derive(s, ctx->stream) != 0 || launch_chi(s, ctx->stream) != 0) {
            rc = fail(ctx, CFUST_ECUDA, cudaGetErrorString(cudaGetLastError()));
            break;
        }
        ctx->launches += 4 + (s.M > 0 ? 1 : 0);   // (+ the lattice sort for the chi nodes)
        // Multi-rank: the communicator is created BEFORE the validation verdict, and the status word
        // (non-finite y, derive errors) is max-reduced over ranks, so every rank returns the same
        // code — a rank failing alone would leave the others blocked in the next collective.
        if (ctx->world > 1 && !opts->nccl_id) { rc = fail(ctx, CFUST_EINVAL, "world > 1 needs nccl_id"); break; }
        if (opts->nccl_id) {   // (world = 1 with an id: a one-rank communicator, every collective path live)
            ncclUniqueId id;
            std::memcpy(&id, opts->nccl_id, sizeof(id));
            ncclResult_t r = ncclCommInitRank(&ctx->comm, ctx->world, id, ctx->rank);
            if (r != ncclSuccess) { rc = fail(ctx, CFUST_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)); break; }
            rc = global_status(ctx);
            if (rc != CFUST_OK) break;
        }
        rc = fetch_status_and_sync(ctx);
        if (rc != CFUST_OK) break;
    } while (0);
    if (rc != CFUST_OK) {
        // keep the message retrievable: return a context only on success; print for the caller
        std::fprintf(stderr, "cfust_em_init: %s\n", ctx->err.c_str());
        cfust_destroy(ctx);
        return rc;
    }
    *out = ctx;
    return CFUST_OK;
}

int cfust_set_data(cfust_ctx *ctx, const double *y, int32_t on_device) {
    if (!ctx || !y) return CFUST_EINVAL;
    DevState &s = ctx->s;
    if (on_device && y != s.y) drop_graphs(ctx);   // the graphs hold s.y as a kernel argument
    if (on_device) {
        s.y = y;
    } else {
        if (!ctx->y_owned) CU(cudaMalloc((void **)&ctx->y_owned, sizeof(double) * (s.n > 0 ? s.n * s.p : 1)));
        if (s.n > 0) CU(cudaMemcpyAsync(ctx->y_owned, y, sizeof(double) * s.n * s.p, cudaMemcpyHostToDevice, ctx->stream));
        s.y = ctx->y_owned;
    }
    return CFUST_OK;
}

int cfust_estep(cfust_ctx *ctx, double *loglik_out, double *stats_out) {
    Nvtx nvtx_range("cfust_estep");
    if (!ctx) return CFUST_EINVAL;
    CU(cudaSetDevice(ctx->device));
    DevState &s = ctx->s;
    int rc = reset_status(ctx);
    if (rc) return rc;
    rc = enqueue_estep(ctx, 0);
    if (rc) return rc;
    const size_t len = size_t(s.g) * s.K + 1;
    CU(cudaMemcpyAsync(ctx->h_pin, s.stats, sizeof(double) * (len + 1), cudaMemcpyDeviceToHost, ctx->stream));
    rc = fetch_status_and_sync(ctx, ctx->h_pin + len);   // global underflow flag (all-reduced)
    acc_phase(ctx, 0, 1, 0);
    acc_phase(ctx, 1, 2, 1);
    acc_phase(ctx, 2, 3, 2);
    ctx->have_stats = (rc == CFUST_OK);
    if (rc) return rc;
    if (loglik_out) *loglik_out = ctx->h_pin[len - 1];
    if (stats_out) std::memcpy(stats_out, ctx->h_pin, sizeof(double) * len);
    return CFUST_OK;
}

int cfust_mstep(cfust_ctx *ctx) {
    Nvtx nvtx_range("cfust_mstep");
    if (!ctx) return CFUST_EINVAL;
    if (!ctx->have_stats) return fail(ctx, CFUST_EINVAL, "cfust_mstep needs a preceding cfust_estep");
    CU(cudaSetDevice(ctx->device));
    int rc = reset_status(ctx);
    if (rc) return rc;
    rec(ctx, 3);
    rc = enqueue_mstep(ctx);
    if (rc) return rc;
    rc = fetch_status_and_sync(ctx);
    acc_phase(ctx, 3, 4, 3);
    ctx->have_stats = false;
    return rc;
}

// E-step + M-step (graph 0) and one host sync: l^(k) and the global underflow flag are read from the
// statistics vector (the M-step leaves it unchanged) together with the status word.
int cfust_iterate(cfust_ctx *ctx, double *loglik_out) {
    Nvtx nvtx_range("cfust_iterate");
    if (!ctx) return CFUST_EINVAL;
    CU(cudaSetDevice(ctx->device));
    DevState &s = ctx->s;
    int rc = reset_status(ctx);
    if (rc) return rc;
    rc = enqueue_iteration(ctx, 0);
    if (rc) return rc;
    const size_t len = size_t(s.g) * s.K + 1;
    CU(cudaMemcpyAsync(ctx->h_pin, s.stats + (len - 1), sizeof(double) * 2, cudaMemcpyDeviceToHost, ctx->stream));
    rc = fetch_status_and_sync(ctx, ctx->h_pin + 1);
    if (!use_graphs(ctx)) {
        acc_phase(ctx, 0, 1, 0);
        acc_phase(ctx, 1, 2, 1);
        acc_phase(ctx, 2, 3, 2);
        acc_phase(ctx, 3, 4, 3);
    }
    ctx->have_stats = false;
    if (rc) return rc;
    if (loglik_out) *loglik_out = ctx->h_pin[0];
    return CFUST_OK;
}

int cfust_loglik(cfust_ctx *ctx, double *out) {
    Nvtx nvtx_range("cfust_loglik");
    if (!ctx || !out) return CFUST_EINVAL;
    CU(cudaSetDevice(ctx->device));
    int rc = reset_status(ctx);
    if (rc) return rc;
    rc = enqueue_estep(ctx, 1);
    if (rc) return rc;
    CU(cudaMemcpyAsync(ctx->h_pin, ctx->d_ll, sizeof(double) * 2, cudaMemcpyDeviceToHost, ctx->stream));
    rc = fetch_status_and_sync(ctx, ctx->h_pin + 1);
    if (rc) return rc;
    *out = ctx->h_pin[0];
    return CFUST_OK;
}

int cfust_predict(cfust_ctx *ctx, int32_t *labels_out, double *tau_out, double *loglik_out) {
    Nvtx nvtx_range("cfust_predict");
    if (!ctx) return CFUST_EINVAL;
    DevState &s = ctx->s;
    CU(cudaSetDevice(ctx->device));
    if (!ctx->d_tau) {
        CU(cudaMalloc((void **)&ctx->d_tau, sizeof(double) * size_t(s.n > 0 ? s.n : 1) * s.g));
        CU(cudaMalloc((void **)&ctx->d_lab, sizeof(int32_t) * size_t(s.n > 0 ? s.n : 1)));
    }
    int rc = reset_status(ctx);
    if (rc) return rc;
    s.tau_out = ctx->d_tau;
    s.label_out = ctx->d_lab;
    rc = enqueue_estep(ctx, 1);
    s.tau_out = nullptr;
    s.label_out = nullptr;
    if (rc) return rc;
    CU(cudaMemcpyAsync(ctx->h_pin, ctx->d_ll, sizeof(double) * 2, cudaMemcpyDeviceToHost, ctx->stream));
    if (labels_out && s.n > 0)
        CU(cudaMemcpyAsync(labels_out, ctx->d_lab, sizeof(int32_t) * s.n, cudaMemcpyDeviceToHost, ctx->stream));
    if (tau_out && s.n > 0)
        CU(cudaMemcpyAsync(tau_out, ctx->d_tau, sizeof(double) * s.n * s.g, cudaMemcpyDeviceToHost, ctx->stream));
    rc = fetch_status_and_sync(ctx, ctx->h_pin + 1);
    if (rc) return rc;
    if (loglik_out) *loglik_out = ctx->h_pin[0];
    return CFUST_OK;
}

static int aitken_stop(double l2, double l1, double l0, double tol) {
    const double den = l1 - l2;
    if (std::fabs(den) < 1e-300) return 1;
    const double a = (l0 - l1) / den;
    if (a >= 1.0) return 0;
    const double linf = l1 + (l0 - l1) / (1.0 - a);
    return std::fabs(linf - l0) < tol;
}

namespace {
// Final l^(K) of a fit: the density-only pass (T0 alone: the same l as the statistics pass of the
// analytic estimator, same kernel split and reduction) — the SOV-direct estimator runs its own
// instantiation for statistics, so there the statistics pass is used to keep the l bits identical
// to cfust_estep.  *dst = device address of [l, underflow flag].
int enqueue_final_pass(cfust_ctx *ctx, const double **dst) {
    const int mode = ctx->s.direct ? 0 : 1;
    const int rc = enqueue_estep(ctx, mode);
    *dst = (mode == 1) ? ctx->d_ll : ctx->s.stats + size_t(ctx->s.g) * ctx->s.K;
    return rc;
}

// Copy trace slots [from, to) of the device ring into tr (after a sync).
void drain_trace(cfust_ctx *ctx, std::vector<double> &tr, int from, int to) {
    for (int k = from; k < to; ++k) tr.push_back(ctx->h_trace[k & (TRACE_CAP - 1)]);
}
}  // namespace

// Fit (Alg. 3-4): E-step at Psi^(0), then per iteration k = 1..max_iter the graph [M-step -> chi
// nodes -> E-step at Psi^(k) -> reduce -> all-reduce] (the last one ends in the final pass).  The
// M-step records l^(k-1) into a device trace ring and gates itself on errors, so with tol <= 0 the
// whole fit is enqueued without a host sync (one at the end; one per TRACE_CAP-1 iterations); with
// tol > 0 there is exactly one host sync per iteration (l^(k) for the Aitken rule, Alg. 4).
int cfust_fit(cfust_ctx *ctx, int32_t max_iter, double tol, cfust_result *out) {
    Nvtx nvtx_range("cfust_fit");
    if (!ctx || !out || max_iter < 0) return CFUST_EINVAL;
    if (out->loglik_trace && out->trace_cap < max_iter + 1) return fail(ctx, CFUST_EINVAL, "trace_cap < max_iter + 1");
    CU(cudaSetDevice(ctx->device));
    const auto t0 = std::chrono::steady_clock::now();
    DevState &s = ctx->s;
    const size_t GK = size_t(s.g) * s.K;
    std::vector<double> tr;
    tr.reserve(size_t(max_iter) + 1);
    out->n_iter = 0;
    out->converged = 0;
    ctx->have_stats = false;
    int rc = reset_status(ctx);
    if (rc) return rc;
    int *hf = ctx->h_fitctl;
    hf[0] = 0; hf[1] = -1; hf[2] = 0; hf[3] = 0;
    CU(cudaMemcpyAsync(s.fitctl, hf, sizeof(int) * 4, cudaMemcpyHostToDevice, ctx->stream));
    const double *lsrc = s.stats + GK;   // [l, underflow flag] of the latest pass
    rc = (max_iter == 0) ? enqueue_final_pass(ctx, &lsrc) : enqueue_estep(ctx, 0);
    if (rc) return rc;
    int drained = 0;   // trace slots already copied to tr
    auto sync_read = [&](int upto) -> int {   // one host sync: fit bookkeeping, trace slots, l, status
        CU(cudaMemcpyAsync(ctx->h_pin, lsrc, sizeof(double) * 2, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaMemcpyAsync(hf, s.fitctl, sizeof(int) * 4, cudaMemcpyDeviceToHost, ctx->stream));
        for (int a = drained; a < upto;) {   // new ring slots only (at most two contiguous pieces)
            const int off = a & (TRACE_CAP - 1), cnt = std::min(upto - a, TRACE_CAP - off);
            CU(cudaMemcpyAsync(ctx->h_trace + off, s.trace + off, sizeof(double) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
            a += cnt;
        }
        CU(cudaMemcpyAsync(ctx->h_status, s.status, sizeof(int) * 4, cudaMemcpyDeviceToHost, ctx->stream));
        const int r = wait_stream(ctx);
        if (r) return r;
        if (upto > drained) { drain_trace(ctx, tr, drained, upto); drained = upto; }
        return CFUST_OK;
    };
    // error bookkeeping -> (rc, n_iter) with orc_fit's semantics: an E-step failure at Psi^(j) ends
    // the fit with n_iter = j - 1; an M-step failure producing Psi^(j+1) with n_iter = j
    auto settle = [&](int k_done) -> int {
        if (hf[1] >= 0) {
            const int j = hf[1];
            out->n_iter = (hf[2] == 1) ? (j > 0 ? j - 1 : 0) : j;
            return check_status(ctx, hf[2] == 1 ? 1.0 : -1.0);
        }
        const int r = check_status(ctx, ctx->h_pin[1]);   // the latest pass (final pass: global flag)
        out->n_iter = (r == CFUST_OK) ? k_done : (k_done > 0 ? k_done - 1 : 0);
        return r;
    };
    double lfinal = 0.0;
    if (max_iter == 0) {
        if ((rc = sync_read(0))) return rc;
        rc = settle(0);
        lfinal = ctx->h_pin[0];
    } else if (tol <= 0.0) {
        for (int k = 1; k <= max_iter && rc == CFUST_OK; ++k) {
            if (k < max_iter) {
                rc = enqueue_iteration(ctx, 1);
            } else {
                rc = enqueue_mstep(ctx);
                if (rc == CFUST_OK) rc = enqueue_final_pass(ctx, &lsrc);
            }
            // the M-step of iteration k wrote slot k-1: drain before the ring wraps
            if (rc == CFUST_OK && k < max_iter && k - drained >= TRACE_CAP - 1) rc = sync_read(k);
        }
        if (rc) return rc;
        if ((rc = sync_read(max_iter))) return rc;
        rc = settle(max_iter);
        lfinal = ctx->h_pin[0];
    } else {
        for (int k = 1; k <= max_iter; ++k) {
            if (k < max_iter) {
                rc = enqueue_iteration(ctx, 1);
            } else {
                rc = enqueue_mstep(ctx);
                if (rc == CFUST_OK) rc = enqueue_final_pass(ctx, &lsrc);
            }
            if (rc) return rc;
            if ((rc = sync_read(k))) return rc;
            if ((rc = settle(k)) != CFUST_OK) break;
            lfinal = ctx->h_pin[0];
            // tr holds l^(0..k-1) (the M-steps' records); with l^(k) from this sync:
            const double lk = lfinal;
            if (k >= 2 && aitken_stop(tr[k - 2], tr[k - 1], lk, tol)) {
                out->converged = 1;
                break;
            }
        }
    }
    // the trace: l^(0..n_iter-1) recorded on the device, l^(n_iter) from the last pass (or the ring)
    const int ni = out->n_iter;
    if (rc == CFUST_OK) {
        tr.resize(size_t(ni));
        tr.push_back(lfinal);
    } else {
        tr.resize(size_t(std::min<int>(int(tr.size()), ni + 1)));
    }
    if (out->loglik_trace)
        for (size_t k = 0; k < tr.size() && int(k) < out->trace_cap; ++k) out->loglik_trace[k] = tr[k];
    out->wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rc;
}

int cfust_get_params(cfust_ctx *ctx, cfust_params *P) {
    if (!ctx || !P || !P->pi || !P->mu || !P->sigma || !P->nu) return CFUST_EINVAL;
    DevState &s = ctx->s;
    CU(cudaSetDevice(ctx->device));
    CU(cudaMemcpyAsync(P->pi, s.pi, sizeof(double) * s.g, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(P->mu, s.mu, sizeof(double) * s.g * s.p, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(P->sigma, s.sigma, sizeof(double) * s.g * s.p * s.p, cudaMemcpyDeviceToHost, ctx->stream));
    if (s.q > 0 && P->delta)
        CU(cudaMemcpyAsync(P->delta, s.delta, sizeof(double) * s.g * s.p * s.q, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(P->nu, s.nu, sizeof(double) * s.g, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return CFUST_OK;
}

int cfust_set_params(cfust_ctx *ctx, const cfust_params *P) {
    if (!ctx) return CFUST_EINVAL;
    DevState &s = ctx->s;
    int rc = validate_params(ctx, s.p, s.q, s.g, P);
    if (rc) return rc;
    CU(cudaSetDevice(ctx->device));
    rc = reset_status(ctx);
    if (rc) return rc;
    rc = upload_params(ctx, P);
    if (rc) return rc;
    CUI(launch_derive(s, ctx->stream));
    CUI(launch_chi(s, ctx->stream));
    ctx->launches += 2;
    ctx->have_stats = false;
    return fetch_status_and_sync(ctx);
}

int cfust_get_pairs(cfust_ctx *ctx, const int64_t *idx, int64_t cnt, double *out) {
    if (!ctx || cnt < 0 || (cnt > 0 && (!idx || !out))) return CFUST_EINVAL;
    if (cnt == 0) return CFUST_OK;
    DevState &s = ctx->s;
    for (int64_t k = 0; k < cnt; ++k)
        if (idx[k] < 0 || idx[k] >= s.n) return fail(ctx, CFUST_EINVAL, "pair index out of range");
    CU(cudaSetDevice(ctx->device));
    const size_t PW = size_t(4 + s.q + s.q * s.q);
    int64_t *d_idx = nullptr;
    double *d_out = nullptr;
    CU(cudaMalloc((void **)&d_idx, sizeof(int64_t) * cnt));
    if (cudaMalloc((void **)&d_out, sizeof(double) * cnt * s.g * PW) != cudaSuccess) {
        cudaFree(d_idx);
        return fail(ctx, CFUST_ECUDA, "cudaMalloc pair_out");
    }
    int rc = reset_status(ctx);
    int nb = 0;
    if (!rc && cudaMemcpyAsync(d_idx, idx, sizeof(int64_t) * cnt, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess)
        rc = fail(ctx, CFUST_ECUDA, "copy idx");
    if (!rc && launch_estep(s, 2, d_idx, cnt, d_out, ctx->stream, &nb) != 0)
        rc = fail(ctx, CFUST_ECUDA, cudaGetErrorString(cudaGetLastError()));
    ctx->launches += 1;
    if (!rc && cudaMemcpyAsync(out, d_out, sizeof(double) * cnt * s.g * PW, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess)
        rc = fail(ctx, CFUST_ECUDA, "copy pair_out");
    if (!rc) rc = fetch_status_and_sync(ctx);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(d_idx);
    cudaFree(d_out);
    return rc;
}

int cfust_eval_special(int32_t which, const double *x, double *y, int64_t n, double aux) {
    if (!x || !y || n < 0 || which < 0 || which > 12) return CFUST_EINVAL;
    if (n == 0) return CFUST_OK;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return CFUST_ECUDA;
    if (upload_special_constants() != 0) return CFUST_ECUDA;
    double *dx = nullptr, *dy = nullptr;
    if (cudaMalloc((void **)&dx, sizeof(double) * n) != cudaSuccess) return CFUST_ECUDA;
    if (cudaMalloc((void **)&dy, sizeof(double) * n) != cudaSuccess) { cudaFree(dx); return CFUST_ECUDA; }
    int rc = CFUST_OK;
    if (cudaMemcpy(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice) != cudaSuccess ||
        launch_special(which, dx, dy, n, aux, 0) != 0 ||
        cudaMemcpy(y, dy, sizeof(double) * n, cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = CFUST_ECUDA;
    cudaFree(dx);
    cudaFree(dy);
    return rc;
}

// ------------------------------------------------------------------------------------------
// Alg. 1: parallel multi-start initialisation, readings I1-I4.
namespace {

struct InitWS {
    double *mind, *cent, *ybar, *sums1, *sums2, *scratch, *amax, *gath;
};

constexpr int SCRATCH = 2048 + 2;

InitWS init_ws(cfust_ctx *ctx) {
    const DevState &s = ctx->s;
    InitWS w;
    w.mind = ctx->d_init;
    w.cent = w.mind + (s.n > 0 ? s.n : 1);
    w.ybar = w.cent + GMAX * PMAX;
    w.sums1 = w.ybar + GMAX * PMAX;
    w.sums2 = w.sums1 + GMAX * (PMAX + 1);
    w.scratch = w.sums2 + GMAX * (PMAX * (PMAX + 1) / 2 + PMAX);
    w.amax = w.scratch + 2048;
    w.gath = w.amax + 2;
    return w;
}

int ensure_init_ws(cfust_ctx *ctx, int m) {
    const DevState &s = ctx->s;
    if (!ctx->d_init) {
        const size_t len = size_t(s.n > 0 ? s.n : 1) + 2 * GMAX * PMAX + GMAX * (PMAX + 1) +
                           GMAX * (PMAX * (PMAX + 1) / 2 + PMAX) + SCRATCH + 2 * size_t(ctx->world);
        CU(cudaMalloc((void **)&ctx->d_init, sizeof(double) * len));
        CU(cudaMalloc((void **)&ctx->d_iflag, sizeof(int) * (GMAX + 1)));
        CU(cudaMallocHost((void **)&ctx->h_ipin, sizeof(double) * (64 + 2 * size_t(ctx->world))));
    }
    if (m > ctx->m_cap) {
        cudaFree(ctx->d_labels);
        ctx->d_labels = nullptr;
        CU(cudaMalloc((void **)&ctx->d_labels, sizeof(int32_t) * size_t(m) * (s.n > 0 ? s.n : 1)));
        ctx->m_cap = m;
    }
    return CFUST_OK;
}

int sync_ctx(cfust_ctx *ctx) { return wait_stream(ctx); }

int allreduce_sum(cfust_ctx *ctx, double *buf, size_t len) {
    if (ctx->comm) NC(ncclAllReduce(buf, buf, len, ncclDouble, ncclSum, ctx->comm, ctx->stream));
    return CFUST_OK;
}

// global per-component sums over labels `lab` (pass 1 or 2) into out (device), all ranks
int global_part_sums(cfust_ctx *ctx, const int32_t *lab, const double *ybar, int pass, double *out) {
    const DevState &s = ctx->s;
    const int E = part_sums_width(s.p, s.g, pass);
    const int cap = int(size_t(max_partial_blocks(s)) * (size_t(s.g) * s.K + 1) / size_t(E));
    int nb = 0;
    CUI(launch_part_sums(s.y, s.n, s.p, s.g, lab, ybar, pass, cap < 4 * s.num_sms ? cap : 4 * s.num_sms, s.partials, &nb,
                         ctx->stream));
    CUI(launch_reduce_cols(s.partials, nb, E, E, out, ctx->stream));
    ctx->launches += 2;
    return allreduce_sum(ctx, out, size_t(E));
}

// global argmax of w.mind (ties -> lowest global index) -> (*val, *idx) on the host
int global_argmax(cfust_ctx *ctx, const InitWS &w, double *val, int64_t *idx) {
    const DevState &s = ctx->s;
    CUI(launch_argmax(w.mind, s.n, ctx->j0, w.scratch, w.amax, ctx->stream));
    ctx->launches += 2;
    if (ctx->comm) {
        NC(ncclAllGather(w.amax, w.gath, 2, ncclDouble, ctx->comm, ctx->stream));
        CU(cudaMemcpyAsync(ctx->h_ipin, w.gath, sizeof(double) * 2 * ctx->world, cudaMemcpyDeviceToHost, ctx->stream));
    } else {
        CU(cudaMemcpyAsync(ctx->h_ipin, w.amax, sizeof(double) * 2, cudaMemcpyDeviceToHost, ctx->stream));
    }
    int rc = sync_ctx(ctx);
    if (rc) return rc;
    double bv = -1.0;
    int64_t bi = INT64_MAX;
    for (int r = 0; r < ctx->world; ++r) {
        const double v = ctx->h_ipin[2 * r];
        const int64_t i = int64_t(ctx->h_ipin[2 * r + 1]);
        if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
    }
    *val = bv;
    *idx = bi;
    return CFUST_OK;
}

// centre slot k <- y_{jg} (global index), broadcast from its owner; mind[jg] <- 0 if set_zero
int set_center_from_point(cfust_ctx *ctx, const InitWS &w, int k, int64_t jg, bool zero_mind) {
    const DevState &s = ctx->s;
    double *dst = w.cent + size_t(k) * s.p;
    const bool mine = jg >= ctx->j0 && jg < ctx->j0 + s.n;
    if (mine) {
        CU(cudaMemcpyAsync(dst, s.y + (jg - ctx->j0) * s.p, sizeof(double) * s.p, cudaMemcpyDeviceToDevice, ctx->stream));
        if (zero_mind) CU(cudaMemsetAsync(w.mind + (jg - ctx->j0), 0, sizeof(double), ctx->stream));
    } else {
        CU(cudaMemsetAsync(dst, 0, sizeof(double) * s.p, ctx->stream));
    }
    return allreduce_sum(ctx, dst, size_t(s.p));   // exactly one rank contributes non-zeros
}

uint64_t splitmix64_host(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

int kmeans_partition(cfust_ctx *ctx, uint64_t seed, int iters, int32_t *lab) {
    const DevState &s = ctx->s;
    const InitWS w = init_ws(ctx);
    const int64_t nt = int64_t(s.n_total);
    const int64_t jstar = int64_t(splitmix64_host(seed ^ 0xA5A5A5A5A5A5A5A5ULL) % uint64_t(nt));
    int rc = set_center_from_point(ctx, w, 0, jstar, false);
    if (rc) return rc;
    CUI(launch_mind(s.y, s.n, s.p, w.cent, w.mind, 1, ctx->stream));
    ctx->launches += 1;
    for (int k = 1; k < s.g; ++k) {   // farthest point (reading I2)
        double v;
        int64_t jb;
        if ((rc = global_argmax(ctx, w, &v, &jb))) return rc;
        if ((rc = set_center_from_point(ctx, w, k, jb, false))) return rc;
        CUI(launch_mind(s.y, s.n, s.p, w.cent + size_t(k) * s.p, w.mind, 0, ctx->stream));
        ctx->launches += 1;
    }
    CU(cudaMemsetAsync(lab, 0xFF, sizeof(int32_t) * (s.n > 0 ? s.n : 1), ctx->stream));   // labels -1
    for (int it = 0; it < iters; ++it) {
        int nb = 0;
        CUI(launch_assign(s.y, s.n, s.p, s.g, w.cent, lab, w.mind, s.partials, &nb, ctx->stream));
        CUI(launch_reduce_cols(s.partials, nb, 1, 1, w.amax, ctx->stream));
        ctx->launches += 2;
        if ((rc = allreduce_sum(ctx, w.amax, 1))) return rc;
        CU(cudaMemcpyAsync(ctx->h_ipin, w.amax, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if ((rc = sync_ctx(ctx))) return rc;
        if (ctx->h_ipin[0] == 0.0) break;
        if ((rc = global_part_sums(ctx, lab, nullptr, 1, w.sums1))) return rc;
        CUI(launch_centers(w.sums1, s.p, s.g, w.cent, ctx->d_iflag, ctx->stream));
        ctx->launches += 1;
        int hflag[GMAX];
        CU(cudaMemcpyAsync(hflag, ctx->d_iflag, sizeof(int) * s.g, cudaMemcpyDeviceToHost, ctx->stream));
        if ((rc = sync_ctx(ctx))) return rc;
        for (int i = 0; i < s.g; ++i) {   // empty cluster: re-seed to the farthest point
            if (!hflag[i]) continue;
            double v;
            int64_t jb;
            if ((rc = global_argmax(ctx, w, &v, &jb))) return rc;
            if ((rc = set_center_from_point(ctx, w, i, jb, true))) return rc;
        }
    }
    return CFUST_OK;
}

int random_partition(cfust_ctx *ctx, uint64_t seed, int l, int m, int32_t *lab) {
    const DevState &s = ctx->s;
    const InitWS w = init_ws(ctx);
    for (int attempt = 0; attempt < 1000; ++attempt) {
        CUI(launch_random_labels(lab, s.n, ctx->j0, s.g, seed, int64_t(l) + int64_t(m) * attempt, ctx->stream));
        ctx->launches += 1;
        int rc = global_part_sums(ctx, lab, nullptr, 1, w.sums1);
        if (rc) return rc;
        CU(cudaMemcpyAsync(ctx->h_ipin, w.sums1, sizeof(double) * s.g * (1 + s.p), cudaMemcpyDeviceToHost, ctx->stream));
        if ((rc = sync_ctx(ctx))) return rc;
        bool ok = true;
        for (int i = 0; i < s.g; ++i)
            if (ctx->h_ipin[i * (1 + s.p)] < double(s.p + 1)) ok = false;
        if (ok) return CFUST_OK;
    }
    return fail(ctx, CFUST_EINVAL, "no random partition with >= p+1 members per component in 1000 draws");
}

}  // namespace

int cfust_init_partitions(cfust_ctx *ctx, int32_t m, uint64_t seed, int32_t kmeans_iters, int32_t *labels_out) {
    Nvtx nvtx_range("cfust_init_partitions");
    if (!ctx || m < 1 || kmeans_iters < 0) return CFUST_EINVAL;
    DevState &s = ctx->s;
    if (s.n_total < double(s.g)) return fail(ctx, CFUST_EINVAL, "n_total < g");
    CU(cudaSetDevice(ctx->device));
    int rc = ensure_init_ws(ctx, m);
    if (rc) return rc;
    const size_t nn = size_t(s.n > 0 ? s.n : 1);
    rc = kmeans_partition(ctx, seed, kmeans_iters, ctx->d_labels);
    for (int l = 1; l < m && !rc; ++l) rc = random_partition(ctx, seed, l, m, ctx->d_labels + size_t(l) * nn);
    if (rc) return rc;
    if (labels_out && s.n > 0)
        CU(cudaMemcpyAsync(labels_out, ctx->d_labels, sizeof(int32_t) * size_t(m) * s.n, cudaMemcpyDeviceToHost,
                           ctx->stream));
    return sync_ctx(ctx);
}

int cfust_init_select(cfust_ctx *ctx, int32_t m, const int32_t *labels, int32_t burn_in, double *loglik0_out,
                      int32_t *best_out) {
    Nvtx nvtx_range("cfust_init_select");
    if (!ctx || m < 1 || burn_in < 0) return CFUST_EINVAL;
    DevState &s = ctx->s;
    if (!labels && m > ctx->m_cap) return fail(ctx, CFUST_EINVAL, "no partitions: call cfust_init_partitions first");
    CU(cudaSetDevice(ctx->device));
    int rc = ensure_init_ws(ctx, m);
    if (rc) return rc;
    const size_t nn = size_t(s.n > 0 ? s.n : 1);
    if (labels && s.n > 0)
        CU(cudaMemcpyAsync(ctx->d_labels, labels, sizeof(int32_t) * size_t(m) * s.n, cudaMemcpyHostToDevice, ctx->stream));
    const InitWS w = init_ws(ctx);
    const int p = s.p, q = s.q, g = s.g;
    std::vector<double> bp(size_t(g) * (1 + p + p * p + p * (q > 0 ? q : 1) + 1));
    cfust_params best_params{bp.data(), bp.data() + g, bp.data() + g + g * p, bp.data() + g + g * p + g * p * p,
                             bp.data() + g + g * p + g * p * p + g * p * (q > 0 ? q : 1)};
    int best = -1;
    double best_ll = -INFINITY;
    for (int c = 0; c < m; ++c) {
        double ll = -INFINITY;
        const int32_t *lab = ctx->d_labels + size_t(c) * nn;
        // Psi^(0) from the partition moments (reading I3), on the device
        if ((rc = global_part_sums(ctx, lab, nullptr, 1, w.sums1))) return rc;
        CUI(launch_centers(w.sums1, p, g, w.ybar, ctx->d_iflag, ctx->stream));
        if ((rc = global_part_sums(ctx, lab, w.ybar, 2, w.sums2))) return rc;
        const int one = 1;
        CU(cudaMemcpyAsync(ctx->d_iflag + GMAX, &one, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
        if ((rc = reset_status(ctx))) return rc;
        CUI(launch_partition_params(s, w.sums1, w.sums2, w.ybar, ctx->d_iflag + GMAX, ctx->stream));
        int valid = 0;
        CU(cudaMemcpyAsync(&valid, ctx->d_iflag + GMAX, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        if ((rc = sync_ctx(ctx))) return rc;
        ctx->launches += 2;
        if (valid) {
            CUI(launch_derive(s, ctx->stream));
            CUI(launch_chi(s, ctx->stream));
            ctx->launches += 2;
            int r2 = fetch_status_and_sync(ctx);
            for (int it = 0; it < burn_in && r2 == CFUST_OK; ++it) r2 = cfust_iterate(ctx, nullptr);
            if (r2 == CFUST_OK) r2 = cfust_loglik(ctx, &ll);
            if (r2 == CFUST_ECUDA || r2 == CFUST_ENCCL) return r2;
            if (r2 != CFUST_OK) ll = -INFINITY;   // candidate failed (ENOTPD, EUNDERFLOW, EEMPTY): skipped
        }
        if (loglik0_out) loglik0_out[c] = ll;
        if (ll > best_ll) {   // strict: ties keep the lowest index (reading I4)
            best_ll = ll;
            best = c;
            if ((rc = cfust_get_params(ctx, &best_params))) return rc;
        }
    }
    if (best < 0) return fail(ctx, CFUST_EINVAL, "every initial partition is invalid");
    if (best_out) *best_out = best;
    ctx->err.clear();
    return cfust_set_params(ctx, &best_params);
}

int cfust_get_timing(cfust_ctx *ctx, double *ms, int64_t *counts, int32_t reset) {
    if (!ctx) return CFUST_EINVAL;
    for (int k = 0; k < 4; ++k) {
        if (ms) ms[k] = ctx->ms[k];
        if (counts) counts[k] = ctx->counts[k];
    }
    if (reset)
        for (int k = 0; k < 4; ++k) { ctx->ms[k] = 0; ctx->counts[k] = 0; }
    return CFUST_OK;
}

}  // extern "C"
