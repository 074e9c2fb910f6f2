"""Pins for the oracle's per-pair E-step and E-step reduction.

The strongest pins integrate the GENERATIVE joint of the CFUST latent representation
(BASELINE.json generator): W ~ Gamma(nu/2, nu/2), U | W ~ N_q(0, I/W)
restricted to u > 0 (density 2^q N), Y | u, W ~ N_p(mu + Delta u, Sigma / W).  They use
none of the oracle's derived formulas (c, Lambda, T_q, truncated moments).
"""
import math

import numpy as np
import pytest
import scipy.integrate as si
import scipy.stats as st

import synth


def _lat(orc, M, seed=11, s=6):
    return orc.Lattice(M, synth.lattice_z(M, s), synth.lattice_shift(seed, s))


# ------------------------------------------------------------------------------ q = 1: exact
@pytest.mark.parametrize("p", [1, 2])
def test_pair_q1_vs_generative_quadrature(orc, p):
    """C5: f, e2, e3, e4 at q=1 vs 2-D quadrature over (u, w) of the generative joint."""
    rng = np.random.default_rng(3 + p)
    mu = rng.standard_normal(p)
    A = rng.standard_normal((p, p))
    Sig = A @ A.T + 0.5 * np.eye(p)
    D = rng.uniform(-2, 2, (p, 1))
    nu = 5.5
    Si = np.linalg.inv(Sig)
    ld = np.linalg.slogdet(Sig)[1]

    # composite Gauss-Legendre in (s, v) with w = e^s, u = e^v (smooth, vectorised)
    xg, wg = np.polynomial.legendre.leggauss(40)

    def grid(lo, hi, panels):
        e = np.linspace(lo, hi, panels + 1)
        x = ((e[1:, None] - e[:-1, None]) * (xg[None, :] + 1) / 2 + e[:-1, None]).ravel()
        w = ((e[1:, None] - e[:-1, None]) / 2 * wg[None, :]).ravel()
        return x, w
    s_, ws = grid(-25.0, 6.0, 40)
    v_, wv = grid(-40.0, 4.0, 40)
    W, U = np.exp(s_)[:, None], np.exp(v_)[None, :]
    jac = (ws * np.exp(s_))[:, None] * (wv * np.exp(v_))[None, :]
    for y in [mu + D[:, 0] * 0.9 + 0.2, mu - 1.0, mu + 2.5 * D[:, 0]]:
        r0 = y - mu
        # r' Si r with r = r0 - D u
        a0, a1, a2 = r0 @ Si @ r0, D[:, 0] @ Si @ r0, D[:, 0] @ Si @ D[:, 0]
        qf = a0 - 2 * a1 * U + a2 * U * U
        ly = -0.5 * p * math.log(2 * math.pi) - 0.5 * ld + 0.5 * p * np.log(W) - 0.5 * W * qf
        joint = st.gamma.pdf(W, nu / 2, scale=2 / nu) * 2 * st.norm.pdf(U, 0, 1 / np.sqrt(W)) * np.exp(ly) * jac
        f = joint.sum()
        e2 = (joint * W).sum() / f
        e3 = (joint * W * U).sum() / f
        e4 = (joint * W * U * U).sum() / f
        r = orc.pair(y, mu, Sig, D, nu, None)
        assert abs(math.exp(r["logf"]) / f - 1) < 1e-9
        assert abs(r["e2"] / e2 - 1) < 1e-9
        assert abs(r["e3"][0] / e3 - 1) < 1e-9
        assert abs(r["e4"][0, 0] / e4 - 1) < 1e-9


# ------------------------------------------------------------------------------ q = 2, 3: MC
def _mc_generative(rng, y, mu, Sig, D, nu, N, reps):
    p, q = D.shape
    Si = np.linalg.inv(Sig)
    ld = np.linalg.slogdet(Sig)[1]
    out = []
    for _ in range(reps):
        w = rng.gamma(nu / 2, 2 / nu, N)
        u = np.abs(rng.standard_normal((N, q))) / np.sqrt(w)[:, None]   # prior of u: 2^q N(0, I/w), u>0
        r = y[None, :] - mu[None, :] - u @ D.T
        qf = np.einsum("ni,ij,nj->n", r, Si, r)
        wt = np.exp(0.5 * p * np.log(w) - 0.5 * w * qf - 0.5 * ld - 0.5 * p * np.log(2 * np.pi))
        f = wt.mean()
        out.append((f, (wt * w).mean() / f, (wt[:, None] * w[:, None] * u).mean(0) / f,
                    np.einsum("n,ni,nj->ij", wt * w, u, u) / N / f))
    return out


@pytest.mark.parametrize("p,q", [(2, 2), (3, 3)])
def test_pair_q23_vs_generative_monte_carlo(orc, p, q):
    """C8: E-step moments for q=2,3 vs self-normalised Monte Carlo of the generative joint."""
    rng = np.random.default_rng(5 + q)
    mu = rng.standard_normal(p)
    A = rng.standard_normal((p, p))
    Sig = A @ A.T + 0.5 * np.eye(p)
    D = rng.uniform(-2, 2, (p, q))
    nu = 6.3
    y = mu + D @ np.abs(rng.standard_normal(q)) * 0.8 + 0.3 * rng.standard_normal(p)
    r = orc.pair(y, mu, Sig, D, nu, _lat(orc, 65536))
    acc = _mc_generative(rng, y, mu, Sig, D, nu, 1_000_000, 4)
    for idx, got in [(0, math.exp(r["logf"])), (1, r["e2"]), (2, r["e3"]), (3, r["e4"])]:
        vals = np.array([a[idx] for a in acc])
        m, se = vals.mean(0), vals.std(0, ddof=1) / math.sqrt(len(vals))
        assert np.all(np.abs(got - m) <= 5 * se + 1e-4 * np.abs(m)), (idx, got, m, se)


# ------------------------------------------------------------------------------ special cases
def test_delta_zero_reduces_to_t(orc):
    """C4: Delta = 0 with q >= 1: T_q(0; I) = 2^-q exactly, so f = t_p and e2 = (nu+p)/(nu+d)."""
    p, q, nu = 3, 3, 7.5
    rng = np.random.default_rng(2)
    A = rng.standard_normal((p, p))
    Sig = A @ A.T + np.eye(p)
    mu = rng.standard_normal(p)
    y = rng.standard_normal(p)
    r = orc.pair(y, mu, Sig, np.zeros((p, q)), nu, _lat(orc, 1024))
    ref = st.multivariate_t(loc=mu, shape=Sig, df=nu).logpdf(y)
    assert abs(r["logf"] - ref) < 1e-12
    d = (y - mu) @ np.linalg.solve(Sig, y - mu)
    assert abs(r["e2"] - (nu + p) / (nu + d)) < 1e-13
    r0 = orc.pair(y, mu, Sig, np.zeros((p, 0)), nu, None)           # the q = 0 family
    assert abs(r0["logf"] - ref) < 1e-12 and abs(r0["e2"] - (nu + p) / (nu + d)) < 1e-13


def test_nu_to_infinity_skew_normal(orc):
    """C6: nu -> inf: f -> 2 phi_p(y; mu, Omega) Phi(c / sqrt(Lambda)), e2 -> 1 (q=1, exact T_1)."""
    p = 2
    mu = np.array([0.2, -0.1])
    Sig = np.array([[1.3, 0.4], [0.4, 0.9]])
    D = np.array([[1.2], [-0.7]])
    y = np.array([0.9, -0.6])
    r = orc.pair(y, mu, Sig, D, 1e7, None)
    Om = Sig + D @ D.T
    c = (D.T @ np.linalg.solve(Om, y - mu))[0]
    lam = 1 - (D.T @ np.linalg.solve(Om, D))[0, 0]
    ref = math.log(2) + st.multivariate_normal(mu, Om).logpdf(y) + st.norm.logcdf(c / math.sqrt(lam))
    assert abs(r["logf"] - ref) < 1e-5
    assert abs(r["e2"] - 1) < 1e-5


def test_density_integrates_to_one_p1q1(orc):
    """C7: p = q = 1 density integrates to 1."""
    mu, Sig, D, nu = 0.3, 1.7, 1.4, 5.5
    f = lambda y: math.exp(orc.pair([y], [mu], [[Sig]], [[D]], nu, None)["logf"])
    tot = si.quad(f, -np.inf, np.inf, epsabs=1e-12, epsrel=1e-12, limit=400)[0]
    assert abs(tot - 1) < 1e-9


def test_density_integrates_to_one_p2q2(orc):
    """C7 on a 2-D grid for p = q = 2 (lattice T_2): within QMC + grid error."""
    rng = np.random.default_rng(9)
    p, q, nu = 2, 2, 9.0
    mu = np.zeros(p)
    Sig = np.array([[1.0, 0.3], [0.3, 0.6]])
    D = rng.uniform(-1, 1, (p, q))
    y = np.stack(np.meshgrid(np.linspace(-14, 16, 121), np.linspace(-14, 16, 121)), -1).reshape(-1, 2)
    lat = _lat(orc, 1024)
    params = {"pi": [1.0], "mu": mu[None], "sigma": Sig[None], "delta": D[None], "nu": [nu]}
    out = orc.estep(y, params, q, lat, pairs=True)
    f = np.exp(out["pairs"][:, 0, 0]).reshape(121, 121)
    h = 30 / 120
    tot = si.simpson(si.simpson(f, dx=h), dx=h)
    assert abs(tot - 1) < 3e-3    # tails beyond the box ~1e-3 at nu = 9


# ------------------------------------------------------------------------------ E-step level
def _problem(cfg_id, n):
    cfg = synth.with_n(synth.CONFIGS[cfg_id], n)
    y, init, truth = synth.make_problem(cfg)
    return cfg, y, init


def test_q0_estep_textbook_t_mixture(orc):
    """q = 0 path: log f, tau, e2 and l equal the textbook t-mixture E-step (scipy logpdf)."""
    cfg, y, init = _problem(3, 500)
    out = orc.estep(y, init, 0, None, pairs=True)
    assert out["rc"] == 0
    lf = np.stack([np.log(init["pi"][i]) + st.multivariate_t(loc=init["mu"][i], shape=init["sigma"][i],
                                                             df=init["nu"][i]).logpdf(y)
                   for i in range(cfg.g)], 1)
    lse = np.logaddexp.reduce(lf, axis=1)
    assert np.max(np.abs(out["pairs"][:, :, 0] - lf)) < 1e-10
    assert np.max(np.abs(out["pairs"][:, :, 1] - np.exp(lf - lse[:, None]))) < 1e-12
    assert abs(out["loglik"] - lse.sum()) < 1e-9 * abs(lse.sum())


@pytest.mark.parametrize("cfg_id,n", [(1, 300), (5, 200)])
def test_estep_invariants(orc, cfg_id, n):
    """C9: sum_i tau = 1; e3 > 0; e4 symmetric PSD; e2 e4 - e3 e3' PSD (Cauchy-Schwarz)."""
    cfg, y, init = _problem(cfg_id, n)
    M, z, sh = synth.lattice_inputs(cfg)
    lat = orc.Lattice(M, z, sh)
    out = orc.estep(y, init, cfg.q, lat, pairs=True)
    assert out["rc"] == 0
    P = out["pairs"]
    q = cfg.q
    assert np.max(np.abs(P[:, :, 1].sum(1) - 1)) < 1e-12
    e2, e3, e4 = P[:, :, 3], P[:, :, 4:4 + q], P[:, :, 4 + q:].reshape(n, cfg.g, q, q)
    assert np.max(np.abs(e4 - np.swapaxes(e4, -1, -2))) == 0.0
    # positivity holds for the exact integrals; the lattice rule keeps it wherever the pair
    # carries weight (in far tails, tau ~ 1e-8, E1 = c T2 + S'h is a QMC-level cancellation)
    sel = P[:, :, 1] > 1e-2
    assert sel.sum() >= n
    assert np.all(e3[sel] > 0) and np.all(e2 > 0)
    assert np.min(np.linalg.eigvalsh(e4[sel])) > 0
    cs = e2[..., None, None] * e4 - e3[..., :, None] * e3[..., None, :]
    assert np.min(np.linalg.eigvalsh(cs[sel])) > -1e-10


def test_stats_packing_and_additivity(orc):
    """S0..S7 recomputed from the per-pair dump; and E-step over two blocks summed equals the
    full E-step (partial-sum additivity, Alg. 2)."""
    cfg, y, init = _problem(1, 400)
    M, z, sh = synth.lattice_inputs(cfg)
    lat = orc.Lattice(M, z, sh)
    out = orc.estep(y, init, cfg.q, lat, pairs=True)
    P = out["pairs"]
    p, q, g = cfg.p, cfg.q, cfg.g
    K = synth.k_stats(p, q)
    assert K == orc.k_stats(p, q) and len(out["stats"]) == g * K + 1
    iu = np.triu_indices(p)
    iq = np.triu_indices(q)
    for i in range(g):
        tau, e1me2, e2 = P[:, i, 1], P[:, i, 2], P[:, i, 3]
        e3, e4 = P[:, i, 4:4 + q], P[:, i, 4 + q:].reshape(-1, q, q)
        ref = np.concatenate([[tau.sum(), (tau * e2).sum()], (tau * e2) @ y,
                              np.einsum("n,na,nb->ab", tau * e2, y, y)[iu], tau @ e3,
                              np.einsum("n,nkl->kl", tau, e4)[iq],
                              np.einsum("n,na,nk->ak", tau, y, e3).ravel(), [(tau * e1me2).sum()]])
        got = out["stats"][i * K:(i + 1) * K]
        assert np.max(np.abs(got - ref) / (np.abs(ref) + 1e-300)) < 1e-12
    a = orc.estep(y[:157], init, q, lat)
    b = orc.estep(y[157:], init, q, lat)
    s = a["stats"] + b["stats"]
    assert np.max(np.abs(s - out["stats"]) / np.abs(out["stats"])) < 1e-12


def test_underflow_error(orc):
    """A16 / SPEC.md:312: every component's f underflows at some y -> EUNDERFLOW."""
    params = {"pi": [1.0], "mu": [[0.0]], "sigma": [[[1e-4]]], "delta": [[[5.0]]], "nu": [1000.0]}
    out = orc.estep(np.array([[-1e4]]), params, 1, None)
    assert out["rc"] == orc.EUNDERFLOW


def test_not_pd_error(orc):
    rc, _ = orc.derive(np.array([[1.0, 2.0], [2.0, 1.0]]), np.zeros((2, 1)), 5.0)
    assert rc == orc.ENOTPD


# ------------------------------------------------------------------------------ exact e1 (R2')
def _joint_grid_q1(p, mu, Sig, D, nu, y):
    """2-D quadrature of the generative joint at q = 1: returns f, E[W|y], E[log W|y]."""
    Si = np.linalg.inv(Sig)
    ld = np.linalg.slogdet(Sig)[1]
    xg, wg = np.polynomial.legendre.leggauss(40)

    def grid(lo, hi, panels):
        e = np.linspace(lo, hi, panels + 1)
        x = ((e[1:, None] - e[:-1, None]) * (xg[None, :] + 1) / 2 + e[:-1, None]).ravel()
        w = ((e[1:, None] - e[:-1, None]) / 2 * wg[None, :]).ravel()
        return x, w
    s_, ws = grid(-25.0, 6.0, 40)
    v_, wv = grid(-40.0, 4.0, 40)
    W, U = np.exp(s_)[:, None], np.exp(v_)[None, :]
    jac = (ws * np.exp(s_))[:, None] * (wv * np.exp(v_))[None, :]
    r0 = y - mu
    a0, a1, a2 = r0 @ Si @ r0, D[:, 0] @ Si @ r0, D[:, 0] @ Si @ D[:, 0]
    qf = a0 - 2 * a1 * U + a2 * U * U
    ly = -0.5 * p * math.log(2 * math.pi) - 0.5 * ld + 0.5 * p * np.log(W) - 0.5 * W * qf
    joint = st.gamma.pdf(W, nu / 2, scale=2 / nu) * 2 * st.norm.pdf(U, 0, 1 / np.sqrt(W)) * np.exp(ly) * jac
    f = joint.sum()
    return f, (joint * W).sum() / f, (joint * np.log(W)).sum() / f


@pytest.mark.parametrize("p", [1, 2])
def test_e1_exact_q1_vs_generative_quadrature(orc, p):
    """Exact e1 = E[log W | y] (reading R2') vs 2-D quadrature of the generative joint at q = 1.
    The lattice estimate is a 1-D rule over the chi node (log V is singular as V -> 0), so the
    pin is: error <= 1e-4 at M = 2^16 and shrinking with M; the A5 approximation is >= 30x worse."""
    rng = np.random.default_rng(13 + p)
    mu = rng.standard_normal(p)
    A = rng.standard_normal((p, p))
    Sig = A @ A.T + 0.5 * np.eye(p)
    D = rng.uniform(-2, 2, (p, 1))
    nu = 5.5
    for y in [mu + D[:, 0] * 0.9 + 0.2, mu - 1.0, mu + 2.5 * D[:, 0]]:
        f, e2, e1 = _joint_grid_q1(p, mu, Sig, D, nu, y)
        errs = []
        for M in [1024, 65536]:
            r = orc.pair(y, mu, Sig, D, nu, _lat(orc, M), e1_exact=True)
            assert abs(math.exp(r["logf"]) / f - 1) < 1e-9          # density unchanged (exact T_1)
            assert abs(r["e2"] / e2 - 1) < 1e-9
            errs.append(abs(r["e1me2"] + r["e2"] - e1))
        assert errs[1] < 1e-4 and errs[1] < errs[0], errs
        r1 = orc.pair(y, mu, Sig, D, nu, None)                          # reading A5
        assert abs(r1["e1me2"] + r1["e2"] - e1) > 30 * errs[1]


def test_e1_exact_delta_zero_closed_form(orc):
    """Delta = 0 (q = 3): Phi_q(0; I) = 2^-q is constant on every lattice point, so the exact e1
    is the lattice mean of log V minus log rho -> psi(m0/2) - log(rho/2) (the A5 formula, exact
    here); the lattice error converges with M."""
    import scipy.special as sp
    p, q, nu = 3, 3, 7.5
    rng = np.random.default_rng(2)
    A = rng.standard_normal((p, p))
    Sig = A @ A.T + np.eye(p)
    mu = rng.standard_normal(p)
    y = rng.standard_normal(p)
    d = (y - mu) @ np.linalg.solve(Sig, y - mu)
    ref = sp.digamma((nu + p) / 2) - math.log((nu + d) / 2)
    errs = []
    for M in [1024, 65536]:
        r = orc.pair(y, mu, Sig, np.zeros((p, q)), nu, _lat(orc, M), e1_exact=True)
        errs.append(abs(r["e1me2"] + r["e2"] - ref))
    assert errs[1] < 1e-5 and errs[1] < errs[0] / 4, errs


def test_e1_exact_q2_vs_generative_monte_carlo(orc):
    """Exact e1 at q = 2 vs self-normalised Monte Carlo of E[log W | y] (5 s.e.)."""
    p, q, nu = 2, 2, 6.3
    rng = np.random.default_rng(21)
    mu = rng.standard_normal(p)
    A = rng.standard_normal((p, p))
    Sig = A @ A.T + 0.5 * np.eye(p)
    D = rng.uniform(-2, 2, (p, q))
    y = mu + D @ np.abs(rng.standard_normal(q)) * 0.8 + 0.3 * rng.standard_normal(p)
    r = orc.pair(y, mu, Sig, D, nu, _lat(orc, 65536), e1_exact=True)
    Si = np.linalg.inv(Sig)
    vals = []
    for _ in range(4):
        w = rng.gamma(nu / 2, 2 / nu, 1_000_000)
        u = np.abs(rng.standard_normal((len(w), q))) / np.sqrt(w)[:, None]
        rr = y[None, :] - mu[None, :] - u @ D.T
        wt = np.exp(0.5 * p * np.log(w) - 0.5 * w * np.einsum("ni,ij,nj->n", rr, Si, rr))
        vals.append((wt * np.log(w)).sum() / wt.sum())
    m, se = np.mean(vals), np.std(vals, ddof=1) / 2
    assert abs(r["e1me2"] + r["e2"] - m) <= 5 * se + 1e-4, (r["e1me2"] + r["e2"], m, se)


def test_e1_exact_estep_stats_q0_unchanged(orc):
    """q = 0: the closed form of reading A5 is already exact; the flag changes nothing."""
    cfg = synth.with_n(synth.CONFIGS[3], 500)
    y, init, _ = synth.make_problem(cfg)
    a = orc.estep(y, init, 0, None)
    b = orc.estep(y, init, 0, None, e1_exact=True)
    assert np.array_equal(a["stats"], b["stats"])
