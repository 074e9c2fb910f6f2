"""Reproduce one wide-fuzz case (tests/test_gpu_fuzz.py with CFUST_FUZZ_SEED / index k) and print the
pairs with the largest e4 disagreement together with their tau, log f and standardized bound."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

os.environ.setdefault("CFUST_FUZZ_SEED", "777")
os.environ.setdefault("CFUST_FUZZ_N", "400")
import synth  # noqa: E402
import oracle  # noqa: E402
import paper_2005_06848_b200 as cf  # noqa: E402
from test_gpu_fuzz import _cases  # noqa: E402
from test_gpu_parity import _olat  # noqa: E402

for k in [int(x) for x in sys.argv[1:]]:
    _, p, q, g, M, n, opt = _cases()[k]
    cfg = synth.with_(synth.CONFIGS[1], n=n, p=p, q=q, g=g, M=M, pi_kind="dirichlet2", data_seed=7000 + k,
                      init_seed=8000 + k, lattice_seed=9000 + k)
    y, init, _ = synth.make_problem(cfg)
    lat = synth.lattice_inputs(cfg, e1_exact=opt.get("e1_exact", False), direct=opt.get("estimator") == "direct")
    em = cf.CfustEM(y, g, q, init, lat, **opt)
    got = em.pairs(np.arange(n))
    ref = oracle.estep(y, init, q, _olat(oracle, lat), pairs=True, gaps=True, **opt)["pairs"]
    e4g, e4r = got[..., 4 + q:], ref[..., 4 + q:]
    s4 = np.max(np.abs(e4r), axis=-1)
    err = np.max(np.abs(e4g - e4r), axis=-1) / s4
    idx = np.dstack(np.unravel_index(np.argsort(-err, axis=None)[:4], err.shape))[0]
    print(f"case {k}: p={p} q={q} g={g} n={n} opt={opt}")
    for j, i in idx:
        print(f"  obs {j} comp {i}: e4 rel err {err[j, i]:.2e}  tau {ref[j, i, 1]:.3e}  logf {ref[j, i, 0]:.2f}"
              f"  e3 {ref[j, i, 4:4 + q]}  e4diag {np.diag(ref[j, i, 4 + q:].reshape(q, q))}")
    em.close()
