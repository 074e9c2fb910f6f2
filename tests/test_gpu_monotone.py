"""C11: the EM log-likelihood trajectory is non-decreasing up to the
integration error of the lattice rule, with the slack CALIBRATED from the multi-shift standard
deviation (randomised QMC: the same rank-1 lattice under R independent random shifts) rather than a
fixed relative constant.  Monotone EM: PAPER.md:197-226 (Eq. (3)-(4) and the E-/M-steps).

At every iterate Psi^(k) of the full-size cfg2 fit (n = 1e5, 20 iterations — the fit where round 1
saw a 1.6e-5-relative dip) the density pass is repeated under R = 6 further shifts; sd_k is the
sample standard deviation of l(Psi^(k)) over the shifts.  Each step must satisfy
    l_{k+1} - l_k >= -4 sqrt(sd_k^2 + sd_{k+1}^2),
i.e. any decrease is within four standard errors of the difference of two integrated values."""
import json
import os

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

R_SHIFTS = 6


@pytest.fixture(scope="module")
def cf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_06848_b200 import build as B
    B.build()
    import paper_2005_06848_b200 as m
    return m


def _shifts(seed, s, r):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(r):
        k = rng.integers(0, 1 << 52, size=max(s, 1), dtype=np.int64)
        out.append((2.0 * k.astype(np.float64) + 1.0) / float(1 << 53))   # as synth.lattice_shift
    return out


def test_cfg2_fit_monotone_within_multishift_sd(cf):
    import torch
    cfg = synth.CONFIGS[2]
    y, init, _ = synth.make_problem(cfg)
    yd = torch.from_numpy(y).cuda()
    M, z, sh = synth.lattice_inputs(cfg)
    em = cf.CfustEM(yd, cfg.g, cfg.q, init, (M, z, sh))
    iters = 20
    trace, psis = [], []
    for _ in range(iters):
        psis.append(em.params())
        trace.append(em.iterate())   # l at Psi^(k), then the M-step
    psis.append(em.params())
    trace.append(em.loglik())
    em.close()
    trace = np.array(trace)
    alt = [cf.CfustEM(yd, cfg.g, cfg.q, init, (M, z, s)) for s in _shifts(20260, len(sh), R_SHIFTS)]
    sd = np.zeros(iters + 1)
    for k, psi in enumerate(psis):
        vals = []
        for a in alt:
            a.set_params(psi)
            vals.append(a.loglik())
        sd[k] = np.std(vals, ddof=1)
    for a in alt:
        a.close()
    d = np.diff(trace)
    slack = 4.0 * np.sqrt(sd[:-1] ** 2 + sd[1:] ** 2)
    ratio = np.where(d < 0, -d / slack, 0.0)
    report = {"trace": trace.tolist(), "sd": sd.tolist(), "diff": d.tolist(), "dip_over_slack": ratio.tolist(),
              "max_dip_rel": float(np.max(np.where(d < 0, -d / np.abs(trace[1:]), 0.0))),
              "sd_rel_median": float(np.median(sd / np.abs(trace)))}
    out = os.environ.get("CFUST_MONOTONE_REPORT")
    if out:
        with open(out, "w") as f:
            json.dump(report, f, indent=1)
    assert np.all(sd > 0.0)
    assert np.all(d >= -slack), report
    assert trace[-1] > trace[0]
    # Exact e1 (reading R2'): the nu step is a true CM step of the ECM, so the same fit on the same
    # lattice must be non-decreasing within the integration slack alone.  (Reading A5's e1 is not the
    # conditional expectation, so the default's nu step maximises a slightly different function: its
    # late decreases (~-15 per step here) are systematic, reproduced to 0.2 % with a 4x finer lattice,
    # and absent under exact e1 — profiles/r02u_monotone_variants.log, reading A5.)
    ex = cf.CfustEM(yd, cfg.g, cfg.q, init, synth.lattice_inputs(cfg, e1_exact=True), e1_exact=True)
    tre = np.array([ex.iterate() for _ in range(iters)] + [ex.loglik()])
    ex.close()
    de = np.diff(tre)
    assert np.all(de >= -slack), (de, slack)
