"""Write the oracle's EM fits at full / reduced BASELINE sizes as goldens for the GPU fit-parity
tests (tests/test_gpu_fullsize.py).  Calls ONLY oracle/ and synth/ (the seeded inputs): no value
here comes from the CUDA path.

    python scripts/make_fit_goldens.py NAME [--budget-s S] [--threads T] [--dir D]

NAME is one of GOLDENS below.  The oracle fit is resumable: every iteration is one oracle E-step
+ M-step (Alg. 3) from the parameters saved after the previous one, so a long
fit can be spread over several runs (each writes tests/golden/fit_NAME.partial.json); the trace
convention is the oracle's (l^(k) at Psi^(k); the final l from the E-step at
the last parameters).  Since the oracle's E-step is deterministic (pairs on any number of threads,
sums serial in ascending j), a resumed fit is bit-identical to an uninterrupted orc_fit.
The finished golden (tests/golden/fit_NAME.json) records the final parameters, the l trace, the
wall time and the host it ran on (the cost the VERDICT asks to state).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

# name -> (config id, n or None for BASELINE n, EM iterations)
GOLDENS = {
    "cfg2_full": (2, None, 20),
    "cfg4_n1e4": (4, 10_000, 5),
    "cfg5_n1e4": (5, 10_000, 5),
}
GDIR = os.path.join(ROOT, "tests", "golden")


def cfg_of(name):
    cid, n, iters = GOLDENS[name]
    cfg = synth.CONFIGS[cid]
    if n is not None:
        cfg = synth.with_n(cfg, n)
    return cfg, iters


def _jsonable(params):
    return {k: np.asarray(v, dtype=np.float64).tolist() for k, v in params.items()}


def oracle_sha():
    h = hashlib.sha256()
    for f in ["cfust_oracle.c", "cfust_oracle.h"]:
        with open(os.path.join(ROOT, "oracle", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def run(name, budget_s, threads, gdir=GDIR):
    cfg, iters = cfg_of(name)
    y, init, _ = synth.make_problem(cfg)
    M, z, sh = synth.lattice_inputs(cfg)
    lat = oracle.Lattice(M, z, sh) if M else None
    part = os.path.join(gdir, f"fit_{name}.partial.json")
    final = os.path.join(gdir, f"fit_{name}.json")
    sha = oracle_sha()
    if os.path.exists(part):
        with open(part) as f:
            st = json.load(f)
        assert st["oracle_sha16"] == sha, "oracle changed since the partial fit was started"
        params = {k: np.asarray(v) for k, v in st["params"].items()}
        trace, k0, spent = st["trace"], st["iters_done"], st["cpu_wall_s"]
        hosts = st["hosts"]
    else:
        params = {k: np.asarray(v, dtype=np.float64) for k, v in init.items()}
        trace, k0, spent, hosts = [], 0, 0.0, []
    host = {"cpu": cpu_model(), "threads": threads}
    if host not in hosts:
        hosts.append(host)
    t_start = time.perf_counter()
    k = k0
    while k < iters:
        t0 = time.perf_counter()
        e = oracle.estep(y, params, cfg.q, lat, nthreads=threads)
        assert e["rc"] == 0, e["rc"]
        assert len(trace) == k
        trace.append(e["loglik"])   # l^(k) at Psi^(k)
        rc, params = oracle.mstep(e["stats"], params, cfg.p, cfg.q, cfg.n)
        assert rc == 0, rc
        k += 1
        dt = time.perf_counter() - t0
        print(f"{name}: iteration {k}/{iters} l^({k - 1}) = {trace[-1]:.12f} ({dt:.1f} s)", flush=True)
        spent_now = spent + (time.perf_counter() - t_start)
        state = {"name": name, "config": cfg.name, "n": cfg.n, "iters": iters, "iters_done": k,
                 "trace": trace, "params": _jsonable(params), "oracle_sha16": sha, "cpu_wall_s": spent_now,
                 "hosts": hosts}
        with open(part + ".tmp", "w") as f:
            json.dump(state, f)
        os.replace(part + ".tmp", part)
        if k < iters and time.perf_counter() - t_start + dt > budget_s:
            print(f"{name}: budget reached after iteration {k}; resume later", flush=True)
            return False
    # final l^(K) at Psi^(K)
    e = oracle.estep(y, params, cfg.q, lat, nthreads=threads)
    assert e["rc"] == 0
    trace.append(e["loglik"])
    spent_now = spent + (time.perf_counter() - t_start)
    gold = {"name": name, "config": cfg.name, "n": cfg.n, "p": cfg.p, "q": cfg.q, "g": cfg.g, "M": cfg.M,
            "iters": iters, "trace": trace, "params": _jsonable(params), "oracle_sha16": sha,
            "cpu_wall_s": spent_now, "hosts": hosts,
            "written_by": "scripts/make_fit_goldens.py (oracle/ + synth/ only)"}
    with open(final, "w") as f:
        json.dump(gold, f, indent=1)
    if os.path.exists(part):
        os.remove(part)
    print(f"{name}: done, {spent_now:.0f} s of oracle time -> {final}", flush=True)
    return True


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+", choices=sorted(GOLDENS))
    ap.add_argument("--budget-s", type=float, default=1e9)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--dir", default=GDIR, help="where the partial / final files are read and written")
    a = ap.parse_args()
    oracle.build()
    os.makedirs(a.dir, exist_ok=True)
    for nm in a.names:
        run(nm, a.budget_s, a.threads, a.dir)


if __name__ == "__main__":
    main()
