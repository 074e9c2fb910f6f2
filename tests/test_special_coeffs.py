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
