"""Pins for the oracle's special functions against closed forms and
independent library routines (scipy / mpmath).  Test-only use of scipy/mpmath."""
import math

import mpmath as mp
import numpy as np
import pytest
import scipy.special as sp
import scipy.stats as st

mp.mp.dps = 40


def _rel(a, b, floor=1e-300):
    return abs(a - b) / max(abs(b), floor)


def test_norm_cdf_vs_scipy_including_tails(orc):
    # relative error bound = conditioning of Phi at x (|d log Phi / d log x| ~ x^2) times a few ulp
    for x in [-37.5, -30.0, -12.0, -5.0, -1.3, -1e-3, 0.0, 0.7, 2.5, 8.0, 9.0]:
        assert _rel(orc.norm_cdf(x), float(mp.ncdf(x))) < 5e-16 * (4.0 + x * x)


def _mp_normq(u):
    u = mp.mpf(u)
    z = mp.mpf(float(sp.ndtri(float(u)))) if float(u) > 1e-300 else mp.mpf(-37)
    for _ in range(60):
        z = z - (mp.ncdf(z) - u) / mp.npdf(z)
    return float(z)


@pytest.mark.parametrize("u", [1e-300, 1e-250, 1e-100, 1e-30, 1e-10, 1e-4, 0.02, 0.3, 0.4999, 0.5,
                               0.5001, 0.8, 0.999, 1 - 1e-9, 1 - 2 ** -53])
def test_norm_quantile_vs_mpmath(orc, u):
    z = orc.norm_quantile(u)
    zr = _mp_normq(u)
    assert abs(z - zr) <= 2e-15 * max(1.0, abs(zr))


def test_norm_quantile_special_values(orc):
    assert orc.norm_quantile(0.5) == 0.0
    assert orc.norm_quantile(0.0) == -math.inf
    assert orc.norm_quantile(1.0) == math.inf
    # textbook quantiles
    assert abs(orc.norm_quantile(0.975) - 1.959963984540054) < 1e-14
    assert abs(orc.norm_quantile(0.8413447460685429) - 1.0) < 1e-14


@pytest.mark.parametrize("a", [0.05, 0.55, 1.0, 2.7, 6.15, 14.0, 33.3])
def test_gamma_p_q_vs_scipy(orc, a):
    for x in [1e-6, 0.01, 0.5, a, a + 1.0, 3 * a + 2, 10 * a + 40]:
        assert _rel(orc.gamma_p(a, x), sp.gammainc(a, x)) < 1e-13
        assert _rel(orc.gamma_q(a, x), sp.gammaincc(a, x)) < 1e-13


def test_gamma_p_closed_form_a1(orc):
    # P(1, x) = 1 - exp(-x)
    for x in [1e-8, 0.3, 2.0, 15.0]:
        assert _rel(orc.gamma_p(1.0, x), -math.expm1(-x)) < 1e-14


@pytest.mark.parametrize("m", [1.1, 2.0, 4.7, 9.3, 12.0, 21.5, 36.0])
def test_chi2_quantile_vs_scipy(orc, m):
    for w in [1e-12, 1e-6, 1e-3, 0.1, 0.5, 0.77, 0.99, 1 - 1e-6, 1 - 1e-11]:
        v = orc.chi2_quantile(w, m)
        assert _rel(v, st.chi2.ppf(w, m)) < 2e-13
        # round trip through the oracle's own P / Q at the other branch
        assert _rel(sp.gammainc(0.5 * m, 0.5 * v), w) < 1e-12 or _rel(sp.gammaincc(0.5 * m, 0.5 * v), 1 - w) < 1e-12


def test_chi2_quantile_closed_form_df2(orc):
    # chi^2_2 is exponential(1/2): v = -2 log(1-w)
    for w in [1e-9, 0.2, 0.5, 0.9, 1 - 1e-8]:
        assert _rel(orc.chi2_quantile(w, 2.0), -2.0 * math.log1p(-w)) < 1e-13


@pytest.mark.parametrize("a,b", [(0.5, 0.5), (2.3, 0.5), (0.5, 7.1), (15.0, 0.5), (3.0, 4.0)])
def test_ibeta_vs_scipy(orc, a, b):
    for x in [1e-9, 0.01, 0.3, 0.5, 0.8, 0.999, 1 - 1e-9]:
        ref = float(mp.betainc(a, b, 0, mp.mpf(x), regularized=True))
        assert _rel(orc.ibeta(a, b, x), ref) < 1e-13


def _t_cdf_mp(x, m):
    mm, xx = mp.mpf(m), mp.mpf(x)
    tail = mp.betainc(mm / 2, mp.mpf(1) / 2, 0, mm / (mm + xx * xx), regularized=True) / 2
    return float(tail) if x < 0 else float(1 - tail)


@pytest.mark.parametrize("m", [1.1, 4.5, 9.3, 20.2, 45.0])
def test_t_cdf_vs_mpmath(orc, m):
    for x in [-80.0, -10.0, -3.0, -0.5, -1e-5, 0.3, 2.0, 7.0]:
        assert _rel(orc.t_cdf(x, m), _t_cdf_mp(x, m)) < 5e-14


def test_t_cdf_closed_forms(orc):
    for x in [-50.0, -2.0, -0.1, 0.0, 0.4, 3.0]:
        # Cauchy (m=1): 1/2 + atan(x)/pi ; m=2: 1/2 + x / (2 sqrt(2+x^2))
        assert abs(orc.t_cdf(x, 1.0) - (0.5 + math.atan(x) / math.pi)) < 1e-15
        assert abs(orc.t_cdf(x, 2.0) - (0.5 + x / (2 * math.sqrt(2 + x * x)))) < 1e-15
    assert orc.t_cdf(0.0, 7.3) == 0.5   # SPEC.md:172 symmetry


def test_t1_logpdf_vs_scipy(orc):
    for (x, loc, s2, m) in [(0.0, 0.3, 1.7, 5.5), (-2.0, 1.0, 0.2, 3.1), (4.0, -1.0, 9.0, 40.0)]:
        assert abs(orc.t1_logpdf(x, loc, s2, m) - st.t.logpdf(x, m, loc=loc, scale=math.sqrt(s2))) < 1e-13
    # Cauchy mode: log(1/pi)
    assert abs(orc.t1_logpdf(0.0, 0.0, 1.0, 1.0) - math.log(1 / math.pi)) < 1e-15


def test_digamma(orc):
    g = 0.57721566490153286061
    assert abs(orc.digamma(1.0) + g) < 1e-14
    assert abs(orc.digamma(2.0) - (1 - g)) < 1e-14
    assert abs(orc.digamma(0.5) - (-g - 2 * math.log(2))) < 1e-14
    for x in [0.05, 0.3, 1.46, 2.5, 7.0, 30.0, 500.0]:
        assert abs(orc.digamma(x) - float(mp.digamma(x))) < 1e-14 * max(1, abs(float(mp.digamma(x))))
