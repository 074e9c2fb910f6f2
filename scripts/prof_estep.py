"""Run the E-step on a config (default cfg2) at n observations, for timing / ncu captures.
--full-slice: take the first n rows of the full-size data set instead of regenerating at n.
--em-iters k: run k EM iterations first (parameters as in bench.py after warm-up)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import synth  # noqa: E402
import paper_2005_06848_b200 as cf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=4000)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--full-slice", action="store_true")
ap.add_argument("--em-iters", type=int, default=0)
ap.add_argument("--estimator", default="analytic", choices=["analytic", "direct"])
a = ap.parse_args()
base = synth.CONFIGS[a.config]
if a.full_slice:
    y, init, _ = synth.make_problem(base)
    y = np.ascontiguousarray(y[:a.n])
    cfg = synth.with_n(base, a.n)
else:
    cfg = synth.with_n(base, a.n)
    y, init, _ = synth.make_problem(cfg)
em = cf.CfustEM(y, cfg.g, cfg.q, init, synth.lattice_inputs(cfg, direct=a.estimator == "direct"), timing=True,
                **({"estimator": "direct"} if a.estimator == "direct" else {}))
for _ in range(a.em_iters):
    em.iterate()
em.timing(reset=True)
for _ in range(a.reps):
    ll = em.estep()
ms, cnt = em.timing()
print(f"lib={os.path.basename(cf._native.LIB_PATH)} est={a.estimator} cfg{a.config} n={a.n} slice={a.full_slice} "
      f"em_iters={a.em_iters} loglik={ll:.6f} estep_ms={ms[0] / max(1, cnt[0]):.4f} "
      f"us_per_obs={1e3 * ms[0] / max(1, cnt[0]) / a.n:.3f}")
