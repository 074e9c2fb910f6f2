"""Write a BASELINE config's synthetic problem in the binary layout examples/cfust_fit.c reads:
python examples/write_problem.py --config 1 --n 1000 problem.bin"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("out")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
if a.n:
    cfg = synth.with_n(cfg, a.n)
y, init, _ = synth.make_problem(cfg)
M, z, sh = synth.lattice_inputs(cfg)
with open(a.out, "wb") as f:
    np.array([cfg.n, cfg.p, cfg.q, cfg.g, M, len(z)], dtype="<i4").tofile(f)
    for arr in [y, init["pi"], init["mu"], init["sigma"], init["delta"], init["nu"]]:
        np.ascontiguousarray(np.asarray(arr, dtype="<f8")).tofile(f)
    if M > 0:
        np.ascontiguousarray(np.asarray(z, dtype="<u4")).tofile(f)
        np.ascontiguousarray(np.asarray(sh, dtype="<f8")).tofile(f)
print(a.out, cfg.name, cfg.n)
