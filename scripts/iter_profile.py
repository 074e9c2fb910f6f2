"""Per-iteration wall time of a full-size fit (to separate work changes along the fit from clock
changes): prints iteration, seconds, loglik; run beside an nvidia-smi sampler."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2005_06848_b200 as cf  # noqa: E402
import synth  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 5
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = synth.CONFIGS[c]
y, init, _ = synth.make_problem(cfg)
yd = torch.from_numpy(y).cuda()
em = cf.CfustEM(yd, cfg.g, cfg.q, init, synth.lattice_inputs(cfg))
for k in range(iters):
    t0 = time.perf_counter()
    ll = em.iterate()
    print(f"iter {k} {time.perf_counter() - t0:.3f} s  loglik {ll:.4f}  t={time.time():.1f}", flush=True)
