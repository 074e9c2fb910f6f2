"""Seeded fuzz parity: random (p, q, g, M, n) with p in 1..8, q in 0..6 (q > p included), g in 1..8,
ragged n, each family / estimator / e1 option, through the C ABI against the oracle (per-pair
outputs — every pair, running-bound tolerance and reading A14 ties as tests/test_gpu_parity.py — and
the statistics at 1e-9).  Covers shapes the five
BASELINE configs do not (p = 1, 5, 7; q = 5; q > p; g = 1, 6, 7)."""
import os

import numpy as np
import pytest

import synth
from test_gpu_parity import _olat, check_pairs, compare_stats

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_06848_b200 import build as B
    B.build()
    import paper_2005_06848_b200 as m
    return m


def _cases():
    # CFUST_FUZZ_N / CFUST_FUZZ_SEED widen the sweep for assurance runs (profiles/r01_fuzz_wide.log)
    rng = np.random.default_rng(int(os.environ.get("CFUST_FUZZ_SEED", "20260")))
    out = []
    opts = [{}, {"e1_exact": True}, {"family": "sn"}, {"estimator": "direct"}]
    for k in range(int(os.environ.get("CFUST_FUZZ_N", "40"))):
        p = int(rng.integers(1, 9))
        q = int(rng.integers(0, 7))
        g = int(rng.integers(1, 9))
        M = int(rng.choice([1024, 2048]))
        n = int(rng.integers(17, 70))
        out.append((k, p, q, g, M, n, opts[k % 4]))
    return out


@pytest.mark.parametrize("k,p,q,g,M,n,opt", _cases())
def test_fuzz_parity(cf, orc, k, p, q, g, M, n, opt):
    cfg = synth.with_(synth.CONFIGS[1], n=n, p=p, q=q, g=g, M=M, pi_kind="dirichlet2", data_seed=7000 + k,
                      init_seed=8000 + k, lattice_seed=9000 + k)
    y, init, _ = synth.make_problem(cfg)
    lat = synth.lattice_inputs(cfg, e1_exact=opt.get("e1_exact", False), direct=opt.get("estimator") == "direct")
    em = cf.CfustEM(y, g, q, init, lat, **opt)
    got = em.pairs(np.arange(n))
    check_pairs(orc, got, y, init, q, lat, **opt)
    ref = orc.estep(y, init, q, _olat(orc, lat), **opt)
    assert ref["rc"] == 0
    ll, st = em.estep(want_stats=True)
    compare_stats(st, ref["stats"], p, q, g)
    em.close()
