"""EM log-likelihood trajectory of the full cfg2 fit (n = 1e5, 20 iterations) under variants, to
separate the causes of the late-iteration decrease (C11): the default (reading A5 for e1), exact e1
(reading R2': the nu step a true CM step), a 4x finer lattice (M = 8192: integration error / 2-4),
and the SOV-direct estimator (reading D1).  Prints l_{k+1} - l_k per variant."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2005_06848_b200 as cf  # noqa: E402

base = synth.CONFIGS[2]
y, init, _ = synth.make_problem(base)
yd = torch.from_numpy(y).cuda()
for name, cfg, kw in [("default", base, {}), ("e1_exact", base, {"e1_exact": True}),
                      ("M8192", synth.with_(base, M=8192), {}), ("direct", base, {"estimator": "direct"}),
                      ("M8192_e1_exact", synth.with_(base, M=8192), {"e1_exact": True})]:
    lat = synth.lattice_inputs(cfg, e1_exact=kw.get("e1_exact", False), direct=kw.get("estimator") == "direct")
    em = cf.CfustEM(yd, cfg.g, cfg.q, init, lat, **kw)
    tr = [em.iterate() for _ in range(20)] + [em.loglik()]
    em.close()
    d = np.diff(tr)
    print(json.dumps({"variant": name, "final": tr[-1], "diff": [round(x, 3) for x in d],
                      "sum_negative": float(d[d < 0].sum())}), flush=True)
