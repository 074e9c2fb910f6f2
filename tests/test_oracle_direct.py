"""Pins for the SOV-direct truncated-moment estimator (NEXT-3, reading D1): the moments are
estimated on T0's own SOV points (drawing the last coordinate too) instead of the analytic
reduction to T_{q-1}, T_{q-2}.  Both estimate the same integrals: they must agree within QMC
error and converge together in M; the density is the same lattice rule (bit-identical log f);
q = 1 against the generative-joint quadrature; the skew-normal family too."""
import math

import numpy as np
import pytest

import synth
from test_oracle_estep import _joint_grid_q1


def _lat(orc, M, seed=11, s=7):
    return orc.Lattice(M, synth.lattice_z(M, s), synth.lattice_shift(seed, s))


def _one(orc, y, mu, Sig, D, nu, lat, **kw):
    prm = {"pi": [1.0], "mu": [mu], "sigma": [Sig], "delta": [D], "nu": [nu]}
    out = orc.estep(np.asarray(y, float)[None, :], prm, D.shape[1], lat, pairs=True, **kw)
    assert out["rc"] == 0
    return out["pairs"][0, 0]


def _rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


@pytest.mark.parametrize("p,q,family", [(2, 2, "st"), (3, 3, "st"), (4, 4, "st"), (6, 6, "st"), (3, 3, "sn")])
def test_direct_agrees_with_analytic(orc, p, q, family):
    rng = np.random.default_rng(60 + q)
    mu = rng.standard_normal(p)
    A = rng.standard_normal((p, p))
    Sig = A @ A.T + 0.5 * np.eye(p)
    D = rng.uniform(-2, 2, (p, q))
    y = mu + D @ np.abs(rng.standard_normal(q)) * 0.8 + 0.3 * rng.standard_normal(p)
    errs = []
    for M in [2048, 65536]:
        L = _lat(orc, M)
        a = _one(orc, y, mu, Sig, D, 6.3, L, e1_exact=family == "st", family=family)
        b = _one(orc, y, mu, Sig, D, 6.3, L, estimator="direct", family=family)
        assert a[0] == b[0]                                  # same T0 lattice rule: identical log f
        errs.append(max(_rel(b[2:4], a[2:4]), _rel(b[4:4 + q], a[4:4 + q]), _rel(b[4 + q:], a[4 + q:])))
    assert errs[1] < 1e-4 and errs[1] < errs[0] / 5, errs


def test_direct_q1_vs_generative_quadrature(orc):
    """q = 1: e1, e2, e3, e4 of the direct estimator vs 2-D quadrature of the generative joint."""
    p = 2
    rng = np.random.default_rng(77)
    mu = rng.standard_normal(p)
    A = rng.standard_normal((p, p))
    Sig = A @ A.T + 0.5 * np.eye(p)
    D = rng.uniform(-2, 2, (p, 1))
    nu = 5.5
    for y in [mu + D[:, 0] * 0.9 + 0.2, mu - 1.0]:
        f, e2, e1 = _joint_grid_q1(p, mu, Sig, D, nu, y)
        r = _one(orc, y, mu, Sig, D, nu, _lat(orc, 65536), estimator="direct")
        assert abs(math.exp(r[0]) / f - 1) < 1e-9                   # exact T_1 density
        assert abs(r[3] / e2 - 1) < 1e-4
        assert abs(r[2] + r[3] - e1) < 1e-4
        ref = orc.pair(y, mu, Sig, D, nu, None)                       # analytic q=1 is exact
        assert abs(r[4] / ref["e3"][0] - 1) < 1e-4 and abs(r[5] / ref["e4"][0, 0] - 1) < 1e-4


def test_direct_estep_stats_and_fit(orc):
    """E-step statistics of the direct estimator are close to the analytic ones (cfg2 slice) and
    the fit's l is monotone up to integration error."""
    cfg = synth.with_n(synth.CONFIGS[2], 60)
    y, init, _ = synth.make_problem(cfg)
    M, z, sh = synth.lattice_inputs(cfg, direct=True)
    L = orc.Lattice(M, z, sh)
    a = orc.estep(y, init, cfg.q, L, e1_exact=True)
    b = orc.estep(y, init, cfg.q, L, estimator="direct")
    assert a["loglik"] == b["loglik"]
    assert _rel(b["stats"], a["stats"]) < 2e-3
    cfg1 = synth.with_n(synth.CONFIGS[1], 600)
    y1, i1, _ = synth.make_problem(cfg1)
    M1, z1, s1 = synth.lattice_inputs(cfg1, direct=True)
    res = orc.fit(y1, i1, cfg1.q, orc.Lattice(M1, z1, s1), max_iter=8, estimator="direct")
    assert res["rc"] == 0
    assert np.all(np.diff(res["trace"]) > -1e-6 * np.abs(res["trace"][1:])), res["trace"]
