"""Per-iteration time of the small configs on the product paths (one B200):
  fit     cfust_fit(K, tol=0): K graph-captured iterations, one host sync at the end
  fit_tol cfust_fit(K, tol>0 unreachable): one host sync per iteration (Aitken needs l^(k))
  iterate cfust_iterate: one graph launch + one host sync per call
  eager   cfust_iterate on a timing context (per-phase events, no graph)
Prints one JSON line per config (ms per EM iteration, wall clock over K iterations)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2005_06848_b200 as cf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,3")
ap.add_argument("--iters", type=int, default=200)
a = ap.parse_args()
for cid in [int(c) for c in a.configs.split(",")]:
    cfg = synth.CONFIGS[cid]
    y, init, _ = synth.make_problem(cfg)
    lat = synth.lattice_inputs(cfg)
    if cid != 1:
        import torch
        y = torch.from_numpy(y).cuda()
    out = {"config": cfg.name, "n": cfg.n, "iters": a.iters}
    em = cf.CfustEM(y, cfg.g, cfg.q, init, lat)
    em.fit(5)
    em.set_params(init)
    r = em.fit(a.iters)
    out["fit_ms"] = 1e3 * r["wall_time_s"] / a.iters
    em.set_params(init)
    r = em.fit(a.iters, 1e-300)
    out["fit_tol_ms"] = 1e3 * r["wall_time_s"] / max(1, r["n_iter"])
    em.set_params(init)
    t0 = time.perf_counter()
    for _ in range(a.iters):
        em.iterate()
    out["iterate_ms"] = 1e3 * (time.perf_counter() - t0) / a.iters
    em.close()
    et = cf.CfustEM(y, cfg.g, cfg.q, init, lat, timing=True)
    et.iterate()
    et.timing(reset=True)
    t0 = time.perf_counter()
    for _ in range(a.iters):
        et.iterate()
    out["eager_iterate_ms"] = 1e3 * (time.perf_counter() - t0) / a.iters
    ms, cnt = et.timing()
    out["phase_ms"] = {"estep": ms[0] / cnt[0], "reduce": ms[1] / cnt[1], "mstep_chi": ms[3] / cnt[3]}
    et.close()
    print(json.dumps(out), flush=True)
