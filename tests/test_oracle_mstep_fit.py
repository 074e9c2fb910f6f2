"""Pins for the oracle's M-step, Aitken rule and fit loop.

The M-step is checked against the stationarity conditions of the complete-data Q function
computed DIRECTLY from the per-pair conditional expectations (no packed statistics):
    mu:    sum_j tau [e2 (y - mu) - Delta_old e3] = 0
    Delta: sum_j tau [(y - mu) e3' - Delta e4]    = 0
    Sigma = (1/S0) sum_j tau E[w (y - mu - Delta u)(y - mu - Delta u)']
    nu:    log(nu/2) - psi(nu/2) + 1 + sum tau (e1 - e2) / sum tau = 0   (or a clamp)
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.special as sp

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _setup(orc, cfg_id, n):
    cfg = synth.with_n(synth.CONFIGS[cfg_id], n)
    y, init, _ = synth.make_problem(cfg)
    M, z, sh = synth.lattice_inputs(cfg)
    lat = orc.Lattice(M, z, sh) if M else None
    return cfg, y, init, lat


@pytest.mark.parametrize("cfg_id,n", [(1, 400), (3, 2000), (5, 150)])
def test_mstep_stationarity(orc, cfg_id, n):
    cfg, y, init, lat = _setup(orc, cfg_id, n)
    p, q, g = cfg.p, cfg.q, cfg.g
    out = orc.estep(y, init, q, lat, pairs=True)
    rc, new = orc.mstep(out["stats"], init, p, q, n)
    assert rc == 0
    P = out["pairs"]
    for i in range(g):
        tau, e1me2, e2 = P[:, i, 1], P[:, i, 2], P[:, i, 3]
        e3 = P[:, i, 4:4 + q]
        e4 = P[:, i, 4 + q:].reshape(-1, q, q) if q else None
        mu, D, Sig = new["mu"][i], new["delta"][i], new["sigma"][i]
        Dold = np.asarray(init["delta"][i]).reshape(p, q)
        r = y - mu
        g_mu = (tau * e2) @ r - Dold @ (tau @ e3) if q else (tau * e2) @ r
        assert np.max(np.abs(g_mu)) < 1e-10 * (1 + np.max(np.abs(tau * e2) @ np.abs(y)))
        if q:
            g_D = np.einsum("n,na,nk->ak", tau, r, e3) - D @ np.einsum("n,nkl->kl", tau, e4)
            assert np.max(np.abs(g_D)) < 1e-9 * (1 + np.abs(np.einsum("n,na,nk->ak", tau, r, e3)).max())
        Ew = (np.einsum("n,na,nb->ab", tau * e2, r, r))
        if q:
            rE3 = np.einsum("n,na,nk->ak", tau, r, e3)
            Ew = Ew - rE3 @ D.T - D @ rE3.T + D @ np.einsum("n,nkl->kl", tau, e4) @ D.T
        Sig_ref = Ew / tau.sum()
        assert np.max(np.abs(Sig - 0.5 * (Sig_ref + Sig_ref.T))) < 1e-10 * np.abs(Sig_ref).max()
        c = (tau * e1me2).sum() / tau.sum()
        nu = new["nu"][i]
        eq = math.log(nu / 2) - sp.digamma(nu / 2) + 1 + c
        if 0.1 < nu < 1000:
            assert abs(eq) < 1e-10
        assert abs(new["pi"][i] - tau.sum() / n) < 1e-12 or new["pi"][i] == pytest.approx(1e-10, rel=0.5)
    assert abs(new["pi"].sum() - 1) < 1e-14


def test_mstep_q_function_increases_each_cm_block(orc):
    """C10: each CM step maximises Q over its block -> random small perturbations decrease Q."""
    cfg, y, init, lat = _setup(orc, 1, 300)
    p, q = cfg.p, cfg.q
    out = orc.estep(y, init, q, lat, pairs=True)
    rc, new = orc.mstep(out["stats"], init, p, q, 300)
    P = out["pairs"]
    i = 0
    tau, e2 = P[:, i, 1], P[:, i, 3]
    e3, e4 = P[:, i, 4:4 + q], P[:, i, 4 + q:].reshape(-1, q, q)

    def Q(mu, D, Sig):
        r = y - mu
        E = (np.einsum("n,na,nb->ab", tau * e2, r, r) - np.einsum("n,na,nk->ak", tau, r, e3) @ D.T
             - D @ np.einsum("n,na,nk->ak", tau, r, e3).T + D @ np.einsum("n,nkl->kl", tau, e4) @ D.T)
        return -0.5 * tau.sum() * np.linalg.slogdet(Sig)[1] - 0.5 * np.trace(np.linalg.solve(Sig, E))
    mu, D, Sig = new["mu"][i], new["delta"][i], new["sigma"][i]
    base = Q(mu, D, Sig)
    rng = np.random.default_rng(0)
    for _ in range(20):
        assert Q(mu, D + 1e-4 * rng.standard_normal(D.shape), Sig) < base   # Delta block (given mu)
        # symmetric perturbation of size 1e-3: Q drops at second order (~1e-6 relative), far above
        # Q's rounding (~1e-16); the earlier 1e-9-sized step sat at the rounding level of Q
        E = 1e-3 * rng.standard_normal((p, p))
        assert Q(mu, D, Sig + 0.5 * (E + E.T)) < base                          # Sigma block


def test_aitken_spec_examples(orc):
    """C14: SPEC.md:341-343 worked sequences (tests/golden/aitken_spec.json) + geometric limit."""
    with open(os.path.join(GOLDEN, "aitken_spec.json")) as f:
        gold = json.load(f)
    for case in gold["cases"]:
        assert orc.aitken_stop(*case["l"], case["eps"]) == (case["decision"] == "stop"), case
    L, c, a = -1234.5, 10.0, 0.7
    l = [L - c * a ** k for k in range(3)]
    # exactly geometric: the extrapolated limit is L, so tol just above |L - l_2| stops
    assert orc.aitken_stop(*l, abs(L - l[2]) * 1.000001)
    assert not orc.aitken_stop(*l, abs(L - l[2]) * 0.999)


def test_fit_loglik_monotone_cfg1(orc):
    """C11: l^(k) non-decreasing along the EM trajectory (cfg1 at full size, 10 iterations)."""
    cfg, y, init, lat = _setup(orc, 1, 1000)
    res = orc.fit(y, init, cfg.q, lat, max_iter=10)
    assert res["rc"] == 0 and res["n_iter"] == 10
    d = np.diff(res["trace"])
    assert np.all(d > -1e-6 * np.abs(res["trace"][1:])), res["trace"]
    assert res["trace"][-1] > res["trace"][0]


def test_fit_monotone_slack_from_multishift_sd(orc):
    """C11 with a calibrated slack (monotone EM): along the
    cfg1 trajectory (n = 1000, 10 iterations) every step satisfies l_{k+1} - l_k >= -4 sqrt(sd_k^2 +
    sd_{k+1}^2), sd_k the standard deviation of l(Psi^(k)) over 6 independent random lattice shifts
    (the integration error of the rule); the slack is also checked to be a small fraction of |l|."""
    cfg, y, init, lat = _setup(orc, 1, 1000)
    M, z, sh = synth.lattice_inputs(cfg)
    rng = np.random.default_rng(20261)
    alts = [orc.Lattice(M, z, (2.0 * rng.integers(0, 1 << 52, size=len(sh)).astype(np.float64) + 1.0) / float(1 << 53))
            for _ in range(6)]
    psi, trace, sd = init, [], []
    for k in range(11):
        ref = orc.estep(y, psi, cfg.q, lat)
        trace.append(ref["loglik"])
        sd.append(np.std([orc.estep(y, psi, cfg.q, a)["loglik"] for a in alts], ddof=1))
        if k < 10:
            res = orc.fit(y, psi, cfg.q, lat, max_iter=1)
            assert res["rc"] == 0
            psi = res["params"]
    trace, sd = np.array(trace), np.array(sd)
    d = np.diff(trace)
    slack = 4.0 * np.sqrt(sd[:-1] ** 2 + sd[1:] ** 2)
    assert np.all(sd > 0.0) and np.all(sd < 1e-5 * np.abs(trace)), sd
    assert np.all(d >= -slack), (d, slack)
    assert trace[-1] > trace[0]


def test_fit_t_mixture_monotone_and_nu_recovery(orc):
    """q=0 (exact EM for the t-mixture): strictly monotone l; nu-hat near 5."""
    cfg = synth.with_(synth.CONFIGS[3], n=10_000, p=2, g=1, nu_lo=5.0, nu_hi=5.0)
    truth = synth.make_truth(cfg)
    y = synth.sample(cfg, truth)
    init = synth.perturb(cfg, truth)
    init["nu"] = np.array([15.0])
    res = orc.fit(y, init, 0, None, max_iter=60, tol=1e-9)
    assert res["rc"] == 0
    assert np.all(np.diff(res["trace"]) > -1e-9 * np.abs(res["trace"][1:]))
    assert 4.0 <= res["params"]["nu"][0] <= 6.5


def test_fit_stops_with_aitken(orc):
    cfg, y, init, lat = _setup(orc, 3, 3000)
    res = orc.fit(y, init, 0, None, max_iter=500, tol=1e-6)
    assert res["converged"] and res["n_iter"] < 500


def test_fit_e1_exact_monotone_and_differs(orc):
    """Exact e1 (reading R2'): the nu step becomes a true CM step of the ECM, so l^(k) is
    non-decreasing up to integration error (cfg1, 10 iterations); the nu estimates differ from
    the reading-A5 fit (the two e1 definitions disagree at the 1e-3 level)."""
    cfg, y, init, lat = _setup(orc, 1, 1000)
    res = orc.fit(y, init, cfg.q, lat, max_iter=10, e1_exact=True)
    assert res["rc"] == 0 and res["n_iter"] == 10
    d = np.diff(res["trace"])
    assert np.all(d > -1e-6 * np.abs(res["trace"][1:])), res["trace"]
    ref = orc.fit(y, init, cfg.q, lat, max_iter=10)
    assert np.max(np.abs(res["params"]["nu"] - ref["params"]["nu"]) / ref["params"]["nu"]) > 1e-4
