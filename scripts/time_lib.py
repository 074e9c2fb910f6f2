"""Time the E-step of an experiment build through the bare C ABI (no binding-level symbol checks):
CFUST_LIB=path python scripts/time_lib.py --config 4 --scale 0.05"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2005_06848_b200._native import Opts, Params  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--scale", type=float, default=0.05)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
L = C.CDLL(os.environ["CFUST_LIB"])
cfg = synth.CONFIGS[a.config]
cfg = synth.with_n(cfg, max(1000, int(cfg.n * a.scale)))
y, init, _ = synth.make_problem(cfg)
M, z, sh = synth.lattice_inputs(cfg)
g, p, q = cfg.g, cfg.p, cfg.q
arrs = [np.ascontiguousarray(np.asarray(init[k], np.float64)) for k in ["pi", "mu", "sigma", "delta", "nu"]]
dp = lambda x: x.ctypes.data_as(C.POINTER(C.c_double))
prm = Params(*[dp(x) for x in arrs])
o = Opts()
zz = np.ascontiguousarray(z, np.uint32)
ss = np.ascontiguousarray(sh, np.float64)
o.lattice_m, o.lattice_z, o.lattice_shift = M, zz.ctypes.data_as(C.POINTER(C.c_uint32)), dp(ss)
o.device, o.world, o.timing = -1, 1, 1
ctx = C.c_void_p()
yy = np.ascontiguousarray(y)
rc = L.cfust_em_init(C.byref(ctx), dp(yy), C.c_int64(len(y)), p, g, q, C.byref(prm), C.byref(o))
assert rc == 0, rc
ll = C.c_double()
L.cfust_estep(ctx, C.byref(ll), None)
ms = np.zeros(4)
cnt = np.zeros(4, np.int64)
L.cfust_get_timing(ctx, dp(ms), cnt.ctypes.data_as(C.POINTER(C.c_int64)), 1)
for _ in range(a.reps):
    L.cfust_estep(ctx, C.byref(ll), None)
L.cfust_get_timing(ctx, dp(ms), cnt.ctypes.data_as(C.POINTER(C.c_int64)), 1)
print(f"lib={os.path.basename(os.environ['CFUST_LIB'])} cfg{a.config} n={cfg.n} loglik={ll.value:.6f} estep_ms={ms[0] / cnt[0]:.3f}")
L.cfust_destroy(ctx)
