"""bench.py — FM-CFUST EM hot path on B200 (arXiv 2005.06848), driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

One "step" = one EM iteration over the whole workload: the E-step kernel (all pairs, all
T_r integrals, truncated moments, tau, the eight sufficient statistics), the deterministic
reduction, the NCCL all-reduce when N > 1, and the device M-step (+ derive + chi nodes).
Workload: BASELINE.json configs[1] (cfg2: n=1e5, p=q=4, g=3, M=2048), synthetic data from
synth/ (the paper's AIS data are not available).  Observations are sharded in
contiguous blocks over ranks (strong scaling of one fit: total work fixed).

Metric: (observation x component) pairs per second of E-step+M-step = n*g / t_iter, plus EM
iterations/s, FP64 roofline fraction of the E-step kernel, and the oracle's CPU rate.
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

METRIC = "CFUST E-step (obs·component)/s and EM iters/s at 1/2/4/8 B200, % FP64 peak"
UNIT = "(obs·component)/s"
# FP64 peak for the "alu" roofline: 148 SMs x 64 DFMA/clk x 2 flop x 1.965 GHz (max SM clock,
# B200_PROFILING.md / MEASURED_PEAKS.json sm_max_mhz).  A DFMA-chain microbenchmark measured on
# the same box is reported beside it (fp64_peak_measured_tflops).
FP64_PEAK_NOMINAL_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
# Executed FP64 flops of the E-step kernel per (obs, component) pair at cfg2, from the ncu
# counters 2*dfma + dadd + dmul over one full-size cfg2 E-step launch (n=1e5, 300000 pairs):
# profiles/r01m_ncu_estep_cfg2_full.txt, re-confirmed in r01n.  Re-measured whenever the kernel changes
# (1.1417e7 with the (10,11) Mills rational, Taylor-13 exp and two-Newton division, r01h).
FP64_FLOPS_PER_PAIR = {2: 9.985e6}
# dram__bytes_read.sum + dram__bytes_write.sum of the same launch: 3.631 MB + 0 B
# (profiles/r01m_ncu_estep_cfg2_full.txt).  Algorithmic bytes: y = 3.2 MB (+ node tables).
TRAFFIC_BYTES_PER_LAUNCH = {2: 3.631e6}
# sm__pipe_fp64_cycles_active (pct of peak, elapsed) of the same launch: the FP64 pipe's busy share,
# which also counts DMUL/DADD/DSETP issue (one flop or none each) — the utilisation view beside the
# flop-rate fraction (profiles/r01n_ncu_estep_cfg2_full.txt).
FP64_PIPE_ACTIVE_NCU = {2: 0.659}


def env_rank():
    r = int(os.environ.get("RANK", "0"))
    w = int(os.environ.get("WORLD_SIZE", "1"))
    lr = int(os.environ.get("LOCAL_RANK", str(r)))
    return r, w, lr


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


def sov_evals_per_pair(q: int) -> int:
    """Normal CDF + quantile evaluations per lattice point per pair (chi-normal SOV):
    T_r costs r Phi + (r-1) Phi^-1 for r >= 2; 2 T_q + q T_{q-1} + C(q,2) T_{q-2}."""
    def cost(r):
        return 2 * r - 1 if r >= 2 else 0
    return 2 * cost(q) + q * cost(q - 1) + (q * (q - 1) // 2) * cost(q - 2)


def cpu_baseline(cfg, y, init, budget_s=15.0):
    """The oracle as it stands, on a bounded strided sample of the workload (rank 0, N=1)."""
    import oracle
    oracle.build()
    M, z, sh = synth.lattice_inputs(cfg)
    lat = oracle.Lattice(M, z, sh) if M else None
    cores = os.cpu_count() or 1
    # calibrate on a tiny sample, then size the sample to ~budget_s
    s0 = max(cores, 8)
    t0 = time.perf_counter()
    oracle.estep(y[:: max(1, len(y) // s0)][:s0], init, cfg.q, lat, nthreads=cores)
    dt = max(time.perf_counter() - t0, 1e-3)
    ns = int(min(len(y), max(s0, s0 * budget_s / dt)))
    sub = y[:: max(1, len(y) // ns)][:ns]
    t0 = time.perf_counter()
    out = oracle.estep(sub, init, cfg.q, lat, nthreads=cores)
    t = time.perf_counter() - t0
    assert out["rc"] == 0
    return {"value": len(sub) * cfg.g / t, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"oracle E-step on a strided sample of {len(sub)} of {len(y)} observations x {cfg.g} "
                      f"components ({t:.1f} s, {cores} OpenMP threads)"}


def run_reference(args, cfg):
    """--impl reference: the CPU oracle on bounded samples of the same workload."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    import oracle
    oracle.build()
    y, init, _ = synth.make_problem(cfg)
    M, z, sh = synth.lattice_inputs(cfg)
    lat = oracle.Lattice(M, z, sh) if M else None
    cores = os.cpu_count() or 1
    # one step = oracle E-step + M-step on a strided sample sized for ~10 s per step
    t0 = time.perf_counter()
    oracle.estep(y[:cores * 2], init, cfg.q, lat, nthreads=cores)
    dt = max(time.perf_counter() - t0, 1e-3)
    ns = int(min(len(y), max(cores * 2, cores * 2 * 8.0 / dt)))
    sub = np.ascontiguousarray(y[:: max(1, len(y) // ns)][:ns])
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
            "warmup": args.warmup, "ms_per_step": tm * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg.name, "n": cfg.n, "p": cfg.p, "q": cfg.q, "g": cfg.g, "M": cfg.M,
                       "sample_n": len(sub)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"oracle E+M step on a strided sample of {len(sub)} observations"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=0, help="override n (testing only; not a bench line)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    if args.n:
        cfg = synth.with_n(cfg, args.n)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist
    import paper_2005_06848_b200 as cf

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    y, init, _ = synth.make_problem(cfg)
    j0, j1 = synth.shard_range(cfg.n, rank, world)
    yl = np.ascontiguousarray(y[j0:j1])
    M, z, sh = synth.lattice_inputs(cfg)
    nccl_id = None
    if world > 1:
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(cf.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy().tobytes())
    yd = torch.from_numpy(yl).cuda()   # inputs resident in HBM before the timed region
    em = cf.CfustEM(yd, cfg.g, cfg.q, init, (M, z, sh), n_total=cfg.n, rank=rank, world=world, nccl_id=nccl_id,
                    device=local, timing=True)
    stream = torch.cuda.ExternalStream(em.stream_ptr)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 256 MB > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        em.iterate()
    em.timing(reset=True)
    l0 = em.launch_count
    step_ms = []
    barrier()
    with ClockSampler(local) as clk:
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
    barrier()
    launches = em.launch_count - l0
    phase_ms, phase_cnt = em.timing(reset=True)
    t_step = float(np.mean(step_ms))
    if world > 1:
        tt = torch.tensor([t_step], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
    value = cfg.n * cfg.g / (t_step * 1e-3)

    # e2e through the public API with HOST buffers: H2D of this rank's y from pinned memory,
    # EM iteration, D2H of the log-likelihood (inside cfust_iterate) — every step.
    pinned = torch.from_numpy(yl).pin_memory()
    yh = pinned.numpy()
    em_h = cf.CfustEM(yh, cfg.g, cfg.q, init, (M, z, sh), n_total=cfg.n, rank=rank, world=world,
                      nccl_id=nccl_id_e2e(world, rank, cf, dist) if world > 1 else None,
                      device=local)
    for _ in range(max(1, args.warmup)):
        em_h.set_data(yh)
        em_h.iterate()
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        em_h.set_data(yh)
        em_h.iterate()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    t_e2e = float(np.mean(e2e_ms))
    if world > 1:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    em_h.close()

    # NEXT rows on the same workload, one GPU only: the driver's multi-GPU runs time
    # the main EM step; the options' multi-rank paths use the same all-reduce pattern
    next_rows = bench_options(cf, cfg, yd, init, (M, z, sh), local,
                              phase_ms[0] / max(1, phase_cnt[0])) if world == 1 else {}

    est_ms = phase_ms[0] / max(1, phase_cnt[0])
    pairs_local = (j1 - j0) * cfg.g
    evals = sov_evals_per_pair(cfg.q) * cfg.M * pairs_local
    fpp = FP64_FLOPS_PER_PAIR.get(args.config)
    peak_meas = measure_fp64_peak()
    roof = {"bound": "alu", "unit": "TFLOP/s", "peak": FP64_PEAK_NOMINAL_TFLOPS,
            "peak_kind": "nominal FP64 (148 SM x 64 DFMA/clk x 2 x 1.965 GHz)",
            "fp64_peak_measured_tflops": peak_meas,
            "traffic": TRAFFIC_BYTES_PER_LAUNCH.get(args.config) if args.n == 0 else None,
            "traffic_unit": "bytes per E-step launch (ncu dram read+write)",
            "kernel": "estep_cfust_kernel", "kernel_ms": est_ms,
            "sov_evals_per_s": evals / (est_ms * 1e-3)}
    if fpp:
        ach = fpp * pairs_local / (est_ms * 1e-3) / 1e12
        roof.update({"achieved": ach, "frac": ach / FP64_PEAK_NOMINAL_TFLOPS,
                     "flops_per_pair": fpp, "fp64_pipe_active_ncu": FP64_PIPE_ACTIVE_NCU.get(args.config)})
    else:
        roof.update({"achieved": None, "frac": None})
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "n": cfg.n, "p": cfg.p, "q": cfg.q, "g": cfg.g, "M": cfg.M,
                       "parallelism": f"dp{world}", "l2": "flushed between timed steps (256 MB write)"},
            "em_iters_per_s": 1e3 / t_step,
            "phase_ms": {"estep": est_ms, "reduce": phase_ms[1] / max(1, phase_cnt[1]),
                         "allreduce": phase_ms[2] / max(1, phase_cnt[2]),
                         "mstep": phase_ms[3] / max(1, phase_cnt[3])},
            "roofline": roof,
            "e2e": {"value": cfg.n * cfg.g / (t_e2e * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": int(yl.nbytes), "d2h_bytes_per_step": 8 + 16},
            "gpu_launches": int(launches),
            "next_rows": next_rows,
            "clocks": clk.summary()}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, y, init)
    if rank == 0:
        print(json.dumps(line), flush=True)
    em.close()
    if world > 1:
        dist.destroy_process_group()


def bench_options(cf, cfg, yd, init, lat, device, default_est_ms):
    """E-step kernel time of each option on the bench workload (one GPU, device-resident y):
    exact e1 (NEXT-2), skew-normal family and SOV-direct moments (NEXT-3), and Alg. 1 multi-start
    initialisation with m = 8 candidates (NEXT-1)."""
    import torch
    rows = {}
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

    if cfg.q >= 1:
        t = estep_ms(e1_exact=True)
        rows["e1_exact"] = {"estep_ms": t, "pairs_per_s": pairs / (t * 1e-3), "overhead_vs_default": t / default_est_ms - 1}
        t = estep_ms(estimator="direct")
        rows["sov_direct"] = {"estep_ms": t, "pairs_per_s": pairs / (t * 1e-3), "speedup_vs_default": default_est_ms / t}
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


def nccl_id_e2e(world, rank, cf, dist):
    import torch
    idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        idt.copy_(torch.frombuffer(bytearray(cf.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(idt, 0)
    return bytes(idt.cpu().numpy().tobytes())


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
