"""CPU check of the CUDA path's fitted Phi / Phi^{-1} (csrc/cfust_special.cuh + cfust_coeffs.h):
the same formulas evaluated in numpy double against mpmath, over the whole range the SOV loop
uses (including region boundaries and tails down to 1e-300).  The device code itself is covered
by the GPU parity tests; this pins the coefficient table and the region logic."""
import os
import re

import mpmath as mp
import numpy as np
import pytest
import scipy.special as sp

mp.mp.dps = 40
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _coeffs():
    txt = open(os.path.join(ROOT, "paper_2005_06848_b200", "csrc", "cfust_coeffs.h")).read()
    return {m.group(1): np.array([float(v) for v in m.group(2).split(",")])
            for m in re.finditer(r"static const double h_(\w+)\[\d+\] = \{([^}]*)\}", txt)}


C = _coeffs()


def horner(c, x):
    r = c[-1]
    for v in c[-2::-1]:
        r = r * x + v
    return r


def phi_emul(x):
    ax = min(abs(x), 40.0)
    hi = ax * ax
    lo = float(mp.mpf(ax) * ax - hi)
    e = np.exp(-0.5 * hi) * (1.0 - 0.5 * lo)
    t = e * (horner(C["PH_P"], ax) / horner(C["PH_Q"], ax))
    return t if x < 0 else 1.0 - t


def phiinv_emul(u):
    t = min(u, 1.0 - u)
    w = -np.log(2.0 * t)
    v = np.sqrt(w)
    z = w * (horner(C["NI_P"], v) / horner(C["NI_Q"], v))
    return -z if u < 0.5 else z


def test_phi_relative_accuracy():
    # down to Phi ~ 5e-308 (below, results are subnormal on every implementation)
    xs = np.concatenate([np.linspace(-37.5, 8.5, 3001), [-1e-8, 1e-8, 0.0]])
    worst = 0.0
    for x in xs:
        ref = mp.ncdf(x)
        got = phi_emul(float(x))
        err = abs(got - ref) / ref
        # conditioning of Phi at x: relative error of x^2 propagates as ~ x^2 eps
        worst = max(worst, float(err) / (1.0 + 0.5 * x * x))
    assert worst < 2e-15, worst


def test_phiinv_relative_accuracy():
    us = np.concatenate([np.logspace(-300, -1, 1500), np.linspace(0.01, 0.99, 1501),
                         1 - np.logspace(-16, -1, 300), [0.5, 0.5 - 1e-12, 0.5 + 2e-12]])
    worst = 0.0
    for u in us:
        um = mp.mpf(float(u))
        z = mp.mpf(float(sp.ndtri(float(u))))
        for _ in range(8):   # Newton on log Phi in high precision from scipy's start
            z = z - (mp.log(mp.ncdf(z)) - mp.log(um)) * mp.ncdf(z) / mp.npdf(z)
        got = phiinv_emul(float(u))
        worst = max(worst, float(abs(got - z) / max(abs(z), mp.mpf(1e-300))) if abs(z) > 1e-3 else float(abs(got - z)))
    assert worst < 3e-15, worst


@pytest.mark.parametrize("name", ["PH_P", "PH_Q", "NI_P", "NI_Q"])
def test_coefficients_positive(name):
    """Horner on a non-negative variable is cancellation-free only with positive coefficients."""
    assert np.all(C[name] > 0)


def test_extremes():
    assert phi_emul(-1e30) == 0.0 and phi_emul(1e30) == 1.0 and phi_emul(0.0) == 0.5
    assert phiinv_emul(0.5) == 0.0


def _seed_coeffs():
    """the FP32 seed literals of seed_U32 in cfust_special.cuh (numerator, then denominator)."""
    txt = open(os.path.join(ROOT, "paper_2005_06848_b200", "csrc", "cfust_special.cuh")).read()
    body = txt[txt.index("float seed_U32(float v)"):]
    body = body[:body.index("return")]
    p = [float(v) for v in re.findall(r"(?:float p = |fmaf\(p, v, )(-?[0-9.e+-]+)f", body)]
    q = [float(v) for v in re.findall(r"(?:float q = |fmaf\(q, v, )(-?[0-9.e+-]+)f", body)]
    assert len(p) == 9 and len(q) == 9
    return np.array(p[::-1], np.float32), np.array(q[::-1], np.float32)   # ascending powers


def phiinv_seed_emul(u, seed_rel_err=0.0):
    """Phiinv_seed: FP32 seed from w = -log(2t), then the third-order FP64 correction with
    Phi's rational.  seed_rel_err perturbs the seed to check the correction's basin."""
    sp_, sq_ = _seed_coeffs()
    t = min(u, 1.0 - u)
    w = np.float32(max(-np.log(2.0 * t), 0.0))
    v = np.float32(np.sqrt(w))
    p = np.float32(0.0)
    for c in sp_[::-1]:
        p = np.float32(p * v + c)
    q = np.float32(0.0)
    for c in sq_[::-1]:
        q = np.float32(q * v + c)
    ax = min(float(np.float32(w * np.float32(p / q))) * (1.0 + seed_rel_err), 37.5)
    hi = ax * ax
    lo = float(mp.mpf(ax) * ax - hi)
    ep = np.exp(0.5 * hi) * (1.0 + 0.5 * lo)
    R = horner(C["PH_P"], ax) / horner(C["PH_Q"], ax)
    r = 2.5066282746310002 * (t * ep - R)
    x = -ax + r * (1.0 + r * (-0.5 * ax + r * (2.0 * hi + 1.0) / 6.0))
    return x if u < 0.5 else -x


@pytest.mark.parametrize("pert", [0.0, 1e-6, -1e-6])
def test_phiinv_seed_accuracy(pert):
    """relative <= 1e-15 for |z| >= 1, absolute <= 1e-15 below, over the SOV range (u >= 1e-300),
    also with the FP32 seed perturbed by 1e-6 (twice its fitted error)."""
    us = np.concatenate([np.logspace(-300, -1, 600), np.linspace(0.01, 0.99, 601),
                         1 - np.logspace(-16, -1, 200), [0.5, 0.5 - 1e-12, 0.5 + 2e-12]])
    worst = 0.0
    for u in us:
        um = mp.mpf(float(u))
        z = mp.mpf(float(sp.ndtri(float(u))))
        for _ in range(8):
            z = z - (mp.log(mp.ncdf(z)) - mp.log(um)) * mp.ncdf(z) / mp.npdf(z)
        got = phiinv_seed_emul(float(u), pert)
        worst = max(worst, float(abs(got - z) / max(abs(z), 1)))
    assert worst < (1e-15 if pert == 0.0 else 3e-15), worst
