"""bench.py — FM-CFUST EM hot path on B200 (arXiv 2005.06848), driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 5]

One "step" = one EM iteration over the whole workload: the E-step kernel (all pairs, all
T_r integrals, truncated moments, tau, the eight sufficient statistics), the deterministic
reduction, the single NCCL all-reduce when N > 1, and the device M-step (+ derive + chi nodes).
Workload: BASELINE.json configs[4] (cfg5: n = 1e7, p = q = 3, g = 8, M = 2048) — the config the
north_star's 1/2/4/8-GPU scaling target is set on; --config 2 gives the round-1
workload.  Synthetic data from synth/ (the paper's AIS data are not available).
Observations are sharded in contiguous blocks over ranks: strong scaling of one fit.

Metric: (observation x component) pairs per second of the EM iteration = n*g / t_iter, plus EM
iterations/s, the FP64 roofline fraction of the E-step kernel, and the oracle's CPU rate.
Multi-rank plumbing (bootstrap, shards, ncclUniqueId, max over ranks): paper_2005_06848_b200.dist.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2005_06848_b200 import dist as D  # noqa: E402

METRIC = "CFUST E-step (obs·component)/s and EM iters/s at 1/2/4/8 B200, % FP64 peak"
UNIT = "(obs·component)/s"
# FP64 peak for the "alu" roofline: 148 SMs x 64 DFMA/clk x 2 flop x 1.965 GHz (max SM clock,
# B200_PROFILING.md / MEASURED_PEAKS.json sm_max_mhz).  A DFMA-chain microbenchmark measured on
# the same box is reported beside it (fp64_peak_measured_tflops).
FP64_PEAK_NOMINAL_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
# Executed FP64 flops per (obs, component) pair and DRAM bytes per E-step launch of the timed kernel,
# per workload: written by scripts/roofline_constants.py from the committed ncu captures it names
# (2*dfma + dadd + dmul and dram__bytes_read/write of one full-size launch).
ROOFLINE_CONSTANTS = os.path.join(ROOT, "profiles", "roofline_constants.json")


def roofline_constants(name):
    try:
        with open(ROOFLINE_CONSTANTS) as f:
            return json.load(f).get(name)
    except OSError:
        return None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if len(s) > 5 + k and s[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def sov_evals_per_pair(q: int) -> int:
    """Normal CDF + quantile evaluations per lattice point per pair (chi-normal SOV):
    T_r costs r Phi + (r-1) Phi^-1 for r >= 2; 2 T_q + q T_{q-1} + C(q,2) T_{q-2}."""
    def cost(r):
        return 2 * r - 1 if r >= 2 else 0
    return 2 * cost(q) + q * cost(q - 1) + (q * (q - 1) // 2) * cost(q - 2)


def _oracle_sample(oracle, cfg, y, init, cores, budget_s):
    """A strided sample of the workload sized for ~budget_s of oracle E-step on `cores` threads."""
    M, z, sh = synth.lattice_inputs(cfg)
    lat = oracle.Lattice(M, z, sh) if M else None
    s0 = max(cores, 8)
    t0 = time.perf_counter()
    oracle.estep(y[:: max(1, len(y) // s0)][:s0], init, cfg.q, lat, nthreads=cores)
    dt = max(time.perf_counter() - t0, 1e-3)
    ns = int(min(len(y), max(s0, s0 * budget_s / dt)))
    return np.ascontiguousarray(y[:: max(1, len(y) // ns)][:ns]), lat


def cpu_baseline(cfg, y, init, budget_s=15.0):
    """The oracle as it stands, on a bounded strided sample of the workload (rank 0, N=1)."""
    import oracle
    oracle.build()
    cores = os.cpu_count() or 1
    sub, lat = _oracle_sample(oracle, cfg, y, init, cores, budget_s)
    t0 = time.perf_counter()
    out = oracle.estep(sub, init, cfg.q, lat, nthreads=cores)
    t = time.perf_counter() - t0
    assert out["rc"] == 0
    # single-core rate: the same oracle on one thread, a sample sized for ~4 s
    sub1, _ = _oracle_sample(oracle, cfg, y, init, 1, 4.0)
    t0 = time.perf_counter()
    out1 = oracle.estep(sub1, init, cfg.q, lat, nthreads=1)
    t1 = time.perf_counter() - t0
    assert out1["rc"] == 0
    return {"value": len(sub) * cfg.g / t, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": cpu_model(),
            "sample": f"oracle E-step on a strided sample of {len(sub)} of {len(y)} observations x {cfg.g} "
                      f"components ({t:.1f} s, {cores} OpenMP threads)",
            "single_core": {"value": len(sub1) * cfg.g / t1, "unit": UNIT, "cores": 1,
                            "sample": f"{len(sub1)} observations x {cfg.g} components ({t1:.1f} s, 1 thread)"}}


def run_reference(args, cfg):
    """--impl reference: the CPU oracle on bounded samples of the same workload (rank 0 only)."""
    rank, world, _ = D.env_rank()
    if rank != 0:
        return
    import oracle
    oracle.build()
    y, init, _ = synth.make_problem(cfg)
    cores = os.cpu_count() or 1
    # one step = oracle E-step + M-step on a strided sample sized for ~8 s per step
    sub, lat = _oracle_sample(oracle, cfg, y, init, cores, 8.0)
    params = init
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        out = oracle.estep(sub, params, cfg.q, lat, nthreads=cores)
        rc, params = oracle.mstep(out["stats"], params, cfg.p, cfg.q, len(sub))
        t = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(t)
    tm = float(np.mean(times))
    v = len(sub) * cfg.g / tm
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tm * 1e3, "ms_per_step_sd": float(np.std(times)) * 1e3,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg.name, "n": cfg.n, "p": cfg.p, "q": cfg.q, "g": cfg.g, "M": cfg.M,
                       "sample_n": len(sub)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": cpu_model(),
                             "sample": f"oracle E+M step on a strided sample of {len(sub)} observations"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--n", type=int, default=0, help="override n (testing only; not a bench line)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-next-rows", action="store_true")
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    if args.n:
        cfg = synth.with_n(cfg, args.n)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import paper_2005_06848_b200 as cf

    rk = D.bootstrap("nccl")
    y, init, _ = synth.make_problem(cfg)
    j0, j1 = rk.shard(cfg.n)
    yl = np.ascontiguousarray(y[j0:j1])
    M, z, sh = synth.lattice_inputs(cfg)
    yd = torch.from_numpy(yl).cuda()   # inputs resident in HBM before the timed region
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 256 MB > 126 MB L2

    def ctx(timing, ydata):
        return cf.CfustEM(ydata, cfg.g, cfg.q, init, (M, z, sh), n_total=cfg.n, rank=rk.rank, world=rk.world,
                          nccl_id=rk.nccl_id(), device=rk.local, timing=timing, global_offset=j0)

    # Probe the step length: a step of >= 20 ms is timed on the eager path with per-phase CUDA events
    # (the E-step kernel's own duration feeds the roofline; graph vs eager differ by ~10 us); shorter
    # steps on the CUDA-graph path (the product's cfust_iterate), phases from a separate short run.
    em = ctx(False, yd)
    em.iterate()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    em.iterate()
    probe_ms = rk.max((time.perf_counter() - t0) * 1e3)
    long_step = probe_ms >= 20.0
    if long_step:
        em.close()
        em = ctx(True, yd)
    stream = torch.cuda.ExternalStream(em.stream_ptr)

    for _ in range(args.warmup):
        em.iterate()
    em.timing(reset=True)
    l0 = em.launch_count
    step_ms = []
    rk.barrier()
    with ClockSampler(rk.local) as clk:
        for _ in range(args.steps):
            flush.zero_()                       # L2 flush between timed iterations (not timed)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            em.iterate()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
    rk.barrier()
    launches = em.launch_count - l0
    if long_step:
        phase_ms, phase_cnt = em.timing(reset=True)
    else:   # phase split on the eager path (3 iterations, not part of the timed value)
        emt = ctx(True, yd)
        emt.iterate()
        emt.timing(reset=True)
        for _ in range(3):
            emt.iterate()
        phase_ms, phase_cnt = emt.timing(reset=True)
        emt.close()
    t_step = rk.max(float(np.mean(step_ms)))
    sd_step = float(np.std(step_ms))
    value = cfg.n * cfg.g / (t_step * 1e-3)

    # e2e through the public API with HOST buffers: H2D of this rank's y from pinned memory,
    # EM iteration, D2H of the log-likelihood (inside cfust_iterate) — every step.  Long steps:
    # min(K, 3) e2e steps (each is seconds; the copy is < 1 % of it).
    pinned = torch.from_numpy(yl).pin_memory()
    yh = pinned.numpy()
    em_h = ctx(False, yh)
    k_e2e = args.steps if not long_step else min(args.steps, 3)
    for _ in range(1 if long_step else max(1, args.warmup)):
        em_h.set_data(yh)
        em_h.iterate()
    rk.barrier()
    e2e_ms = []
    for _ in range(k_e2e):
        t0 = time.perf_counter()
        em_h.set_data(yh)
        em_h.iterate()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    t_e2e = rk.max(float(np.mean(e2e_ms)))
    em_h.close()

    est_ms = phase_ms[0] / max(1, phase_cnt[0])
    pairs_local = (j1 - j0) * cfg.g
    evals = sov_evals_per_pair(cfg.q) * cfg.M * pairs_local
    rc = roofline_constants(cfg.name) if args.n == 0 else None
    peak_meas = measure_fp64_peak()
    roof = {"bound": "alu", "unit": "TFLOP/s", "peak": FP64_PEAK_NOMINAL_TFLOPS,
            "peak_kind": "nominal FP64 (148 SM x 64 DFMA/clk x 2 x 1.965 GHz)",
            "fp64_peak_measured_tflops": peak_meas,
            "kernel": "estep_cfust_kernel" if cfg.q else "estep_t_mma_kernel", "kernel_ms": est_ms,
            "sov_evals_per_s": evals / (est_ms * 1e-3)}
    if rc:
        ach = rc["flops_per_pair"] * pairs_local / (est_ms * 1e-3) / 1e12
        roof.update({"achieved": ach, "frac": ach / FP64_PEAK_NOMINAL_TFLOPS,
                     "frac_of_measured_peak": ach / peak_meas if peak_meas else None,
                     "flops_per_pair": rc["flops_per_pair"],
                     "traffic": rc["dram_bytes_per_launch"] * (j1 - j0) / cfg.n,
                     "traffic_unit": "bytes per E-step launch (ncu dram read + write, this rank's share)",
                     "traffic_read_write": [rc["dram_read_bytes"], rc["dram_write_bytes"]],
                     "algorithmic_bytes": yl.nbytes,
                     "fp64_pipe_active_ncu": rc.get("fp64_pipe_active"), "source": rc.get("source")})
    else:
        roof.update({"achieved": None, "frac": None, "traffic": None})
    # NEXT rows on one GPU: each option's E-step and Alg. 1 (cfg5: on the first 10^6
    # observations — the options' full-size times are in profiles/ and DESIGN §5)
    next_rows = {}
    if rk.world == 1 and not args.no_next_rows:
        nr = min(cfg.n, 1_000_000)
        next_rows = bench_options(cf, synth.with_n(cfg, nr), yd[:nr], init, (M, z, sh), rk.local)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": rk.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step, "ms_per_step_sd": sd_step,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "n": cfg.n, "p": cfg.p, "q": cfg.q, "g": cfg.g, "M": cfg.M,
                       "parallelism": f"dp{rk.world}", "l2": "flushed between timed steps (256 MB write)",
                       "path": "eager + per-phase events" if long_step else "CUDA graph"},
            "em_iters_per_s": 1e3 / t_step,
            "phase_ms": {"estep": est_ms, "reduce": phase_ms[1] / max(1, phase_cnt[1]),
                         "allreduce": phase_ms[2] / max(1, phase_cnt[2]),
                         "mstep": phase_ms[3] / max(1, phase_cnt[3])},
            "roofline": roof,
            "e2e": {"value": cfg.n * cfg.g / (t_e2e * 1e-3), "unit": UNIT, "steps": k_e2e,
                    "h2d_bytes_per_step": int(yl.nbytes), "d2h_bytes_per_step": 8 + 16},
            "gpu_launches": int(launches),
            "next_rows": next_rows,
            "clocks": clk.summary()}
    if rk.rank == 0 and rk.world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, y, init)
    if rk.rank == 0:
        print(json.dumps(line), flush=True)
    em.close()
    rk.close()


def bench_options(cf, cfg, yd, init, lat, device):
    """E-step kernel time of each option on (a slice of) the bench workload (one GPU, device-resident
    y): exact e1 (NEXT-2), skew-normal family and SOV-direct moments (NEXT-3), the default estimator
    for reference, and Alg. 1 multi-start initialisation with m = 8 candidates (NEXT-1)."""
    import torch
    rows = {"n": cfg.n}
    pairs = cfg.n * cfg.g

    def estep_ms(**kw):
        latk = synth.lattice_inputs(cfg, e1_exact=kw.get("e1_exact", False), direct=kw.get("estimator") == "direct")
        em = cf.CfustEM(yd, cfg.g, cfg.q, init, latk, device=device, timing=True, **kw)
        em.estep()
        em.timing(reset=True)
        for _ in range(2):
            em.estep()
        ms, cnt = em.timing(reset=True)
        em.close()
        return ms[0] / max(1, cnt[0])

    t_def = estep_ms()
    rows["default"] = {"estep_ms": t_def, "pairs_per_s": pairs / (t_def * 1e-3)}
    if cfg.q >= 1:
        t = estep_ms(e1_exact=True)
        rows["e1_exact"] = {"estep_ms": t, "pairs_per_s": pairs / (t * 1e-3), "overhead_vs_default": t / t_def - 1}
        t = estep_ms(estimator="direct")
        rows["sov_direct"] = {"estep_ms": t, "pairs_per_s": pairs / (t * 1e-3), "speedup_vs_default": t_def / t}
    t = estep_ms(family="sn")
    rows["skew_normal"] = {"estep_ms": t, "pairs_per_s": pairs / (t * 1e-3)}
    em = cf.CfustEM(yd, cfg.g, cfg.q, init, lat, device=device)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    em.init_partitions(8, seed=2005, kmeans_iters=50, want_labels=False)
    t1 = time.perf_counter()
    ll0, best = em.init_select(8)
    t2 = time.perf_counter()
    rows["multistart_init"] = {"m": 8, "partitions_ms": (t1 - t0) * 1e3, "select_ms": (t2 - t1) * 1e3,
                               "best": best, "loglik0_best": float(ll0[best])}
    em.close()
    return rows


def measure_fp64_peak():
    import ctypes as C
    from paper_2005_06848_b200 import build as B
    try:
        L = C.CDLL(B.PEAK_LIB)
        L.fp64_peak_tflops.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double)]
        t = C.c_double(0)
        ms = C.c_double(0)
        if L.fp64_peak_tflops(C.byref(t), C.byref(ms)) == 0:
            return t.value
    except OSError:
        pass
    return None


if __name__ == "__main__":
    main()
