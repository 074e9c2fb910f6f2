"""Pins for the oracle's lattice and T_r (readings A11-A15, R-T).

T_r is the chi-normal separation-of-variables rule on the shifted rank-1 lattice.  It is
pinned against: exact lattice arithmetic (integers/fractions), the elliptical orthant
closed forms (any df), 1-D adaptive quadrature for r=2 at general b, the r=1 closed form,
sign symmetry (Delta=0 -> 2^-q exactly), permutation and diagonal-scale invariance of the
reordering, and convergence in M.
"""
from fractions import Fraction

import numpy as np
import pytest
import scipy.integrate as si
import scipy.special as sp
import scipy.stats as st

import synth


def _lat(orc, M, seed=7, s=6):
    return orc.Lattice(M, synth.lattice_z(M, s), synth.lattice_shift(seed, s))


def test_lattice_points_exact(orc):
    M = 1024
    lat = _lat(orc, M)
    z, sh = synth.lattice_z(M, 6), synth.lattice_shift(7, 6)
    for l in [0, 1, 5, 511, 1023]:
        for k in range(6):
            t = (l * int(z[k])) % M
            x = Fraction(t, M) + Fraction(sh[k])
            if x >= 1:
                x -= 1
            ref = abs(2 * x - 1)
            # double rounding of t/M + shift only: within 1 ulp of the exact rational
            assert abs(Fraction(orc.lattice_w(lat, l, k)) - ref) <= Fraction(2, 1 << 53)


def test_lattice_table_properties():
    for M in [1024, 2048, 4096, 8192, 16384, 32768, 65536]:
        z = synth.lattice_z(M, 6)
        assert z[0] == 1 and all(int(v) % 2 == 1 for v in z) and all(0 < int(v) < M // 2 + 1 for v in z)
    sh = synth.lattice_shift(2002, 6)
    assert np.all((sh > 0) & (sh < 1))
    assert np.all(np.mod(sh * 2.0 ** 53, 2.0) == 1.0)    # odd multiples of 2^-53 (A15)


def test_chi_table_vs_scipy(orc):
    lat = _lat(orc, 1024)
    for m in [3.5, 9.2, 26.0]:
        tab = orc.chi_table(lat, m)
        w = np.array([orc.lattice_w(lat, l, 0) for l in range(lat.M)])
        ref = np.sqrt(st.chi2.ppf(w, m) / m)
        assert np.max(np.abs(tab / ref - 1)) < 1e-13


def test_logchi_table_vs_scipy(orc):
    """log V_l = log chi2_m^{-1}(w_l) (exact e1, reading R2') against scipy's quantile, absolute
    error (log V can be ~0)."""
    lat = _lat(orc, 1024)
    for m in [3.5, 9.2, 26.0]:
        lv = orc.logchi_table(lat, m)
        w = np.array([orc.lattice_w(lat, l, 0) for l in range(lat.M)])
        assert np.max(np.abs(lv - np.log(st.chi2.ppf(w, m)))) < 1e-12


def test_Tr_w_consistent_with_Tr(orc):
    """The weighted lattice rule returns the same T as the plain one and, with lv = 1 everywhere,
    wsum = T (the weights enter only the second sum)."""
    import ctypes as C
    lat = _lat(orc, 2048)
    b = np.array([0.3, -0.2, 0.9])
    S = np.array([[1.0, 0.3, 0.1], [0.3, 1.2, -0.2], [0.1, -0.2, 0.8]])
    m = 7.5
    chi = orc.chi_table(lat, m)
    T = orc.Tr(b, S, m, lat, chi)
    ones = np.ones(lat.M)
    ws = np.zeros(1)
    gap = np.array([np.inf])
    Tw = orc.lib().orc_Tr_w(3, orc._p(b), orc._p(S), m, lat.ptr, orc._p(chi), orc._p(ones), orc._p(gap), orc._p(ws))
    assert Tw == T and abs(ws[0] - T) <= 1e-15


def test_T0_T1_closed(orc):
    assert orc.Tr(np.zeros(0), np.zeros((0, 0)), 5.0) == 1.0
    for b, s, m in [(0.4, 2.0, 5.3), (-3.0, 0.7, 11.0)]:
        assert abs(orc.Tr([b], [[s]], m) - sp.stdtr(m, b / np.sqrt(s))) < 1e-14


@pytest.mark.parametrize("M,tol2,tol3", [(1024, 5e-6, 2e-5), (4096, 5e-6, 1e-5)])
def test_orthant_closed_forms(orc, M, tol2, tol3):
    """C2: T_2(0) = 1/4 + asin(rho)/(2 pi), T_3(0) = 1/8 + sum asin(rho_kl)/(4 pi), any df."""
    lat = _lat(orc, M)
    S = np.array([[1.0, 0.6], [0.6, 2.0]])
    rho = 0.6 / np.sqrt(2.0)
    for m in [4.3, 7.3, 30.0]:
        assert abs(orc.Tr([0, 0], S, m, lat) - (0.25 + np.arcsin(rho) / (2 * np.pi))) < tol2
    S3 = np.array([[1, 0.3, -0.2], [0.3, 1.5, 0.4], [-0.2, 0.4, 0.8]])
    D = np.sqrt(np.diag(S3))
    R = S3 / np.outer(D, D)
    ex = 1 / 8 + (np.arcsin(R[0, 1]) + np.arcsin(R[0, 2]) + np.arcsin(R[1, 2])) / (4 * np.pi)
    assert abs(orc.Tr([0, 0, 0], S3, 5.5, lat) - ex) < tol3


def test_sign_symmetry_identity_scale_exact(orc):
    """C4: T_q(0; 0, I, m) = 2^-q exactly for every lattice point (each SOV factor is Phi(0))."""
    lat = _lat(orc, 2048)
    for q in [2, 3, 4, 6]:
        assert orc.Tr(np.zeros(q), np.eye(q), 6.7, lat) == 2.0 ** -q


def _T2_quad(b, S, m):
    s11 = S[0, 0]

    def f(x):
        mu = S[1, 0] / s11 * x
        sc2 = (m + x * x / s11) / (m + 1) * (S[1, 1] - S[1, 0] ** 2 / s11)
        return st.t.pdf(x, m, scale=np.sqrt(s11)) * sp.stdtr(m + 1, (b[1] - mu) / np.sqrt(sc2))
    return si.quad(f, -np.inf, b[0], epsabs=1e-14, epsrel=1e-13, limit=500)[0]


def test_T2_general_b_vs_quadrature(orc):
    """C3: brute-force 1-D quadrature of t_1(x) T_{m+1}(conditional) for r = 2."""
    S = np.array([[1.0, 0.6], [0.6, 2.0]])
    lat = _lat(orc, 65536)
    for b, m in [((0.7, -0.4), 6.2), ((-2.5, 1.0), 4.5), ((3.0, 3.0), 9.0), ((-0.3, -1.2), 14.0)]:
        b = np.array(b)
        ref = _T2_quad(b, S, m)
        assert abs(orc.Tr(b, S, m, lat) / ref - 1) < 1e-6


def test_T_convergence_in_M(orc):
    S = np.array([[1.0, 0.6], [0.6, 2.0]])
    b, m = np.array([-2.5, 1.0]), 4.5
    ref = _T2_quad(b, S, m)
    errs = [abs(orc.Tr(b, S, m, _lat(orc, M)) / ref - 1) for M in [1024, 16384, 65536]]
    assert errs[2] < errs[0] and errs[2] < 1e-6


def test_reordering_permutation_and_scale_invariance(orc):
    """A13: keys b_k/sqrt(S_kk) sorted ascending -> any input permutation or positive diagonal
    rescaling gives the same integral (to rounding)."""
    lat = _lat(orc, 2048)
    rng = np.random.default_rng(1)
    for q in [3, 4, 6]:
        A = rng.standard_normal((q, q))
        S = A @ A.T + q * np.eye(q)
        b = rng.standard_normal(q)
        m = 8.1
        v = orc.Tr(b, S, m, lat)
        P = rng.permutation(q)
        assert abs(orc.Tr(b[P], S[np.ix_(P, P)], m, lat) - v) < 1e-14
        D = np.exp(rng.standard_normal(q))
        assert abs(orc.Tr(D * b, S * np.outer(D, D), m, lat) / v - 1) < 1e-12


def test_T3_vs_scipy_mvt(orc):
    """Cross-check against scipy's own (randomised QMC) multivariate t CDF at r = 3."""
    lat = _lat(orc, 65536)
    S3 = np.array([[1, 0.3, -0.2], [0.3, 1.5, 0.4], [-0.2, 0.4, 0.8]])
    b = np.array([0.5, -0.3, 1.1])
    m = 6.0
    ref = st.multivariate_t(loc=np.zeros(3), shape=S3, df=m).cdf(b, maxpts=4_000_000, random_state=3)
    assert abs(orc.Tr(b, S3, m, lat) / ref - 1) < 2e-3


def test_monotone_and_limits(orc):
    lat = _lat(orc, 2048)
    S = np.array([[1.0, -0.4, 0.2], [-0.4, 1.0, 0.1], [0.2, 0.1, 1.0]])
    m = 5.0
    v0 = orc.Tr([0.1, 0.2, -0.3], S, m, lat)
    v1 = orc.Tr([0.1, 0.5, -0.3], S, m, lat)
    assert v1 > v0
    assert orc.Tr([60, 60, 60], S, m, lat) > 1 - 1e-6
    assert orc.Tr([60, -1e4, 60], S, m, lat) < 1e-12
