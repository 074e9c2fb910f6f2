"""Pins for the skew-normal family (CFUSN, nu = inf; NEXT-3, reading F1) and its q = 0 case, the
Gaussian mixture: scipy's normal / skew-normal densities and
truncated-normal moments, generative Monte Carlo, the nu -> inf limit of the skew-t oracle, and
scikit-learn's Gaussian-mixture EM step."""
import math

import numpy as np
import pytest
import scipy.stats as st

import synth


def _lat(orc, M, seed=11, s=6):
    return orc.Lattice(M, synth.lattice_z(M, s), synth.lattice_shift(seed, s))


def test_gaussian_component_density(orc):
    p = 4
    rng = np.random.default_rng(0)
    A = rng.standard_normal((p, p))
    Sig = A @ A.T + np.eye(p)
    mu, y = rng.standard_normal(p), rng.standard_normal(p)
    r = orc.pair(y, mu, Sig, np.zeros((p, 0)), 5.0, None, family="sn")
    assert abs(r["logf"] - st.multivariate_normal(mu, Sig).logpdf(y)) < 1e-12
    assert r["e2"] == 1.0 and r["e1me2"] == 0.0


def test_skew_normal_p1_density_and_moments(orc):
    """p = q = 1: f = scipy skewnorm(a = delta/sigma, loc = mu, scale = sqrt(sigma^2 + delta^2));
    e3, e4 = first two moments of N(c, Lambda) truncated to (0, inf) (scipy truncnorm)."""
    mu, sig2, dl = 0.4, 1.3, -1.7
    om = math.sqrt(sig2 + dl * dl)
    for y in [-2.0, 0.1, 1.9]:
        r = orc.pair([y], [mu], [[sig2]], [[dl]], 7.0, None, family="sn")
        ref = st.skewnorm(dl / math.sqrt(sig2), loc=mu, scale=om).logpdf(y)
        assert abs(r["logf"] - ref) < 1e-12
        c = dl * (y - mu) / (sig2 + dl * dl)
        lam = 1 - dl * dl / (sig2 + dl * dl)
        tn = st.truncnorm((0 - c) / math.sqrt(lam), np.inf, loc=c, scale=math.sqrt(lam))
        assert abs(r["e3"][0] / tn.mean() - 1) < 1e-12
        assert abs(r["e4"][0, 0] / tn.moment(2) - 1) < 1e-11


@pytest.mark.parametrize("p,q", [(2, 2), (3, 3)])
def test_skew_normal_q23_vs_generative_monte_carlo(orc, p, q):
    """W = 1: u ~ |N(0, I)|, y | u ~ N(mu + Delta u, Sigma); f, E[u|y], E[u u'|y] by MC (5 s.e.)."""
    rng = np.random.default_rng(40 + q)
    mu = rng.standard_normal(p)
    A = rng.standard_normal((p, p))
    Sig = A @ A.T + 0.5 * np.eye(p)
    D = rng.uniform(-2, 2, (p, q))
    y = mu + D @ np.abs(rng.standard_normal(q)) * 0.8 + 0.3 * rng.standard_normal(p)
    r = orc.pair(y, mu, Sig, D, 3.0, _lat(orc, 65536), family="sn")
    Si = np.linalg.inv(Sig)
    ld = np.linalg.slogdet(Sig)[1]
    vals = []
    for _ in range(4):
        u = np.abs(rng.standard_normal((1_000_000, q)))
        rr = y[None, :] - mu[None, :] - u @ D.T
        wt = np.exp(-0.5 * np.einsum("ni,ij,nj->n", rr, Si, rr) - 0.5 * ld - 0.5 * p * math.log(2 * math.pi))
        f = wt.mean()
        vals.append((f, (wt[:, None] * u).mean(0) / f, np.einsum("n,ni,nj->ij", wt, u, u) / len(wt) / f))
    for idx, got in [(0, math.exp(r["logf"])), (1, r["e3"]), (2, r["e4"])]:
        v = np.array([a[idx] for a in vals])
        m, se = v.mean(0), v.std(0, ddof=1) / 2
        assert np.all(np.abs(got - m) <= 5 * se + 1e-4 * np.abs(m)), (idx, got, m, se)


def test_skew_t_limit_is_skew_normal(orc):
    """nu -> inf: the skew-t pair (chi radius -> 1) tends to the skew-normal pair, O(1/nu)."""
    p, q = 3, 3
    rng = np.random.default_rng(8)
    mu = rng.standard_normal(p)
    A = rng.standard_normal((p, p))
    Sig = A @ A.T + np.eye(p)
    D = rng.uniform(-1.5, 1.5, (p, q))
    y = mu + 0.5 * rng.standard_normal(p)
    lat = _lat(orc, 1024)
    errs = []
    for nu in [1e4, 1e6]:
        a = orc.pair(y, mu, Sig, D, nu, lat)
        b = orc.pair(y, mu, Sig, D, nu, lat, family="sn")
        errs.append(max(abs(a["logf"] - b["logf"]), abs(a["e2"] - 1), np.max(np.abs(a["e3"] - b["e3"])),
                        np.max(np.abs(a["e4"] - b["e4"]))))
    assert errs[1] < 1e-4 and errs[1] < errs[0] / 20, errs   # O(1/nu) convergence


def test_gaussian_mixture_em_step_vs_sklearn(orc):
    """q = 0, family "sn": one E+M step equals scikit-learn GaussianMixture's first EM iteration
    from the same start (weights, means, precisions; reg_covar = 0)."""
    from sklearn.mixture import GaussianMixture
    cfg = synth.with_(synth.with_n(synth.CONFIGS[3], 3000), p=3, g=3)
    y, init, _ = synth.make_problem(cfg)
    st_ = orc.estep(y, init, 0, None, family="sn")
    rc, P = orc.mstep(st_["stats"], init, cfg.p, 0, len(y), family="sn")
    assert rc == 0 and np.array_equal(P["nu"], np.asarray(init["nu"]))   # nu untouched
    gm = GaussianMixture(cfg.g, covariance_type="full", reg_covar=0.0, max_iter=1, tol=0.0,
                         weights_init=init["pi"], means_init=init["mu"],
                         precisions_init=np.linalg.inv(init["sigma"]))
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        gm.fit(y)
    assert np.allclose(P["pi"], gm.weights_, rtol=1e-10)
    assert np.allclose(P["mu"], gm.means_, rtol=1e-10, atol=1e-12)
    assert np.allclose(P["sigma"], gm.covariances_, rtol=1e-9, atol=1e-12)


def test_skew_normal_fit_monotone(orc):
    """CFUSN EM is an exact EM (no e1 approximation): l non-decreasing along the fit."""
    cfg = synth.with_n(synth.CONFIGS[1], 1000)
    y, init, _ = synth.make_problem(cfg)
    M, z, sh = synth.lattice_inputs(cfg)
    res = orc.fit(y, init, cfg.q, orc.Lattice(M, z, sh), max_iter=10, family="sn")
    assert res["rc"] == 0
    assert np.all(np.diff(res["trace"]) > -1e-7 * np.abs(res["trace"][1:])), res["trace"]
