"""Device special functions (the code the E-step kernels inline), through the C ABI diagnostic
cfust_eval_special, against mpmath / scipy.  Tolerances include the conditioning of each
function at its argument."""
import mpmath as mp
import numpy as np
import pytest
import scipy.special as sp
import scipy.stats as st

pytestmark = pytest.mark.gpu
mp.mp.dps = 40


@pytest.fixture(scope="module")
def cf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_06848_b200 import build as B
    B.build()
    import paper_2005_06848_b200 as m
    return m


@pytest.mark.parametrize("name", ["phi", "phi_xt"])
def test_phi(cf, name):
    x = np.concatenate([np.linspace(-37.5, 8.5, 20001), [0.0, -1e-300, 1e-300, -45.0, 45.0, -1e30, 1e30]])
    y = cf.eval_special(name, x)
    ref = np.array([float(mp.ncdf(v)) for v in x])
    ok = np.abs(x) <= 37.5
    rel = np.abs(y[ok] - ref[ok]) / ref[ok] / (1.0 + 0.5 * x[ok] ** 2)
    assert rel.max() < 2e-15, rel.max()
    assert y[-4] == 0.0 and y[-3] == 1.0 and y[-2] == 0.0 and y[-1] == 1.0


@pytest.mark.parametrize("name", ["phiinv", "phiinv_xt"])
def test_phiinv(cf, name):
    u = np.concatenate([np.logspace(-300, -1, 3000), np.linspace(0.001, 0.999, 3001), 1 - np.logspace(-16, -1, 500),
                        [0.5, np.nextafter(0.5, 0), np.nextafter(0.5, 1)]])
    z = cf.eval_special(name, u)
    for ui, zi in zip(u[::7], z[::7]):
        ref = mp.mpf(float(sp.ndtri(ui)))
        for _ in range(6):
            ref = ref - (mp.log(mp.ncdf(ref)) - mp.log(mp.mpf(ui))) * mp.ncdf(ref) / mp.npdf(ref)
        # relative for |z| >= 1, absolute below: the SOV loop consumes z only through the linear
        # form a = s b - sum C z, and near u = 1/2 the seeded correction is exact to ~4e-16 absolute
        err = abs(zi - ref) / max(abs(ref), mp.mpf(1))
        assert err < 3e-15, (ui, zi, ref)
    assert z[-3] == 0.0


def test_exp_table(cf):
    # the SOV loop's optional table exp (CFUST_SOV_XT builds): negative arguments (Phi) and positive ones up to
    # 703 (e^{z0^2/2} of the quantile correction, |z0| <= 37.5)
    x = np.concatenate([-np.logspace(-12, np.log10(708), 5000), np.logspace(-12, np.log10(703.2), 5000), [0.0]])
    y = cf.eval_special("exp_xt", x)
    ref = np.array([float(mp.exp(mp.mpf(float(v)))) for v in x])
    assert np.max(np.abs(y - ref) / ref) < 5e-16
    assert cf.eval_special("exp_xt", np.array([-709.0, -745.0]))[1] == 0.0


def test_exp_log_sqrt(cf):
    x = np.concatenate([-np.logspace(-12, np.log10(708), 5000), [0.0, -1e-300]])
    y = cf.eval_special("exp", x)
    rel = np.abs(y - np.exp(x)) / np.exp(x)
    assert rel.max() < 5e-16
    assert cf.eval_special("exp", np.array([-709.0, -745.0, -1e4]))[2] == 0.0
    u = np.concatenate([np.logspace(-300, 0, 5000), 1 - np.logspace(-16, -1, 1000)])
    lg = cf.eval_special("log", u)
    ref = np.array([float(mp.log(mp.mpf(float(v)))) for v in u])
    ok = ref != 0
    assert np.max(np.abs(lg[ok] - ref[ok]) / np.abs(ref[ok])) < 5e-16
    assert cf.eval_special("log", np.array([1.0]))[0] == 0.0
    w = np.concatenate([np.linspace(0, 700, 5001), np.logspace(-300, 2, 500)])
    s = cf.eval_special("sqrt", w)
    assert np.max(np.abs(s - np.sqrt(w)) / np.maximum(np.sqrt(w), 1e-300)) < 3e-16


@pytest.mark.parametrize("df", [1.3, 5.7, 13.0, 30.5])
def test_t_cdf_chi2_digamma(cf, df):
    x = np.concatenate([np.linspace(-40, 20, 601), [0.0]])
    tc = cf.eval_special("t_cdf", x, df)
    ref = np.array([float(mp.betainc(df / 2, 0.5, 0, df / (df + v * v), regularized=True) / 2) if v < 0 else
                    float(1 - mp.betainc(df / 2, 0.5, 0, df / (df + v * v), regularized=True) / 2) for v in x])
    assert np.max(np.abs(tc - ref) / ref) < 5e-14
    w = np.concatenate([np.logspace(-12, -0.5, 200), 1 - np.logspace(-12, -0.5, 200)])
    q = cf.eval_special("chi2_quantile", w, df)
    assert np.max(np.abs(q / st.chi2.ppf(w, df) - 1)) < 1e-12
    d = cf.eval_special("digamma", np.array([0.05, 0.5, 1.0, 2.5, 10.0, 77.0, df]))
    assert np.max(np.abs(d - sp.digamma([0.05, 0.5, 1.0, 2.5, 10.0, 77.0, df]))) < 1e-13


def test_lgamma_range(cf):
    """log Gamma of the M-step's derived constants (one code path for every argument) vs scipy:
    absolute 1e-14 where |lgamma| <= 1 (Stirling after the recurrence: ~1e-15 cancellation error),
    relative 1e-14 elsewhere, over the df range (nu/2, (nu+p+k)/2)."""
    x = np.concatenate([np.linspace(0.05, 40, 800), np.geomspace(40, 600, 50), [0.5, 1.0, 1.5, 2.0, 2.5, 10.0]])
    got = cf.eval_special("lgamma", x)
    ref = sp.gammaln(x)
    assert np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref))) < 1e-14


def test_trigamma_and_digamma_range(cf):
    """psi and psi' (the M-step's nu equation and its Newton derivative) vs scipy over the nu range."""
    x = np.concatenate([np.linspace(0.05, 40, 800), [0.5, 1.0, 16.0, 100.0, 500.0]])
    tg = cf.eval_special("trigamma", x)
    assert np.max(np.abs(tg / sp.polygamma(1, x) - 1)) < 5e-15
    dg = cf.eval_special("digamma", x)
    assert np.max(np.abs(dg - sp.digamma(x)) / np.maximum(1, np.abs(sp.digamma(x)))) < 2e-15
