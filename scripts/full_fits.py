"""Every BASELINE config at full size for its stated number of EM iterations (BASELINE.json configs:
10 / 20 / 10 / 5 / 5), one GPU, device-resident y: the log-likelihood trace, its monotonicity and
the wall time of the fit (cfust_fit).  -> profiles/r01_full_fits.log"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_06848_b200 as cf  # noqa: E402
import synth  # noqa: E402

cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "1,2,3,4,5").split(",")]
for c in cfgs:
    cfg = synth.CONFIGS[c]
    y, init, _ = synth.make_problem(cfg)
    yd = torch.from_numpy(y).cuda()
    em = cf.CfustEM(yd, cfg.g, cfg.q, init, synth.lattice_inputs(cfg))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = em.fit(cfg.iters)
    wall = time.perf_counter() - t0
    tr = np.asarray(res["trace"])
    d = np.diff(tr)
    print(json.dumps({"config": cfg.name, "n": cfg.n, "p": cfg.p, "q": cfg.q, "g": cfg.g, "M": cfg.M,
                      "em_iters": int(res["n_iter"]), "fit_wall_s": round(wall, 4),
                      "s_per_iter": round(wall / max(1, res["n_iter"]), 5),
                      "loglik_first": float(tr[0]), "loglik_last": float(tr[-1]),
                      "monotone": bool(np.all(d >= -1e-9 * np.abs(tr[1:]))),
                      "min_step": float(d.min()) if len(d) else None,
                      "nu": [round(float(v), 4) for v in res["params"]["nu"]]}), flush=True)
    em.close()
    del yd
    torch.cuda.empty_cache()
