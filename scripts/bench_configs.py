"""Per-config E-step / EM-iteration timing on one GPU (full BASELINE sizes unless --scale < 1).
Prints one JSON line per config: E-step ms, M-step ms, pairs/s, SOV evaluations/s."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2005_06848_b200 as cf  # noqa: E402


def evals_per_pair_point(q):
    c = lambda r: 2 * r - 1 if r >= 2 else 0
    return 2 * c(q) + q * c(q - 1) + (q * (q - 1) // 2) * c(q - 2)


ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3,4,5")
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--estimator", default="analytic", choices=["analytic", "direct"])
ap.add_argument("--family", default="st", choices=["st", "sn"])
ap.add_argument("--e1-exact", action="store_true")
a = ap.parse_args()
for cid in [int(c) for c in a.configs.split(",")]:
    cfg = synth.CONFIGS[cid]
    cfg = synth.with_n(cfg, max(1000, int(cfg.n * a.scale)))
    y, init, _ = synth.make_problem(cfg)
    yd = torch.from_numpy(y).cuda()
    lat = synth.lattice_inputs(cfg, e1_exact=a.e1_exact, direct=a.estimator == "direct")
    em = cf.CfustEM(yd, cfg.g, cfg.q, init, lat, timing=True, estimator=a.estimator, family=a.family,
                    e1_exact=a.e1_exact)
    em.iterate()
    em.timing(reset=True)
    for _ in range(a.iters):
        em.iterate()
    ms, cnt = em.timing()
    est = ms[0] / cnt[0]
    it = sum(ms) / cnt[0]
    pairs = cfg.n * cfg.g
    out = {"config": cfg.name, "estimator": a.estimator, "family": a.family, "e1_exact": a.e1_exact, "n": cfg.n, "p": cfg.p, "q": cfg.q, "g": cfg.g, "M": cfg.M,
           "estep_ms": est, "reduce_ms": ms[1] / cnt[1], "mstep_ms": ms[3] / cnt[3], "iter_ms": it,
           "pairs_per_s": pairs / (it * 1e-3), "em_iters_per_s": 1e3 / it,
           "sov_evals_per_s": pairs * cfg.M * evals_per_pair_point(cfg.q) / (est * 1e-3) if cfg.q >= 2 else None,
           "y_bytes": y.nbytes, "hbm_gbs_estep": y.nbytes / (est * 1e-3) / 1e9}
    print(json.dumps(out), flush=True)
    em.close()
    del yd
    torch.cuda.empty_cache()
