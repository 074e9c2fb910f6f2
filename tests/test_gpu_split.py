"""Small-n statistics pass with SPLIT warps per observation (estep_cfust_kernel<Q, 0, false, SPLIT>):
every forced SPLIT (env CFUST_SPLIT, read at context creation) matches the oracle at the 1e-9
statistics tolerance, and agrees with the one-warp path to rounding (only the order of the lattice
sum changes).  Auto selection (split_factor) is exercised by every small-n parity test."""
import numpy as np
import pytest

from test_gpu_parity import TOL, _olat, _problem, cf, compare_stats  # noqa: F401 (cf: fixture)

pytestmark = pytest.mark.gpu

CASES = [(1, 300), (2, 97), (5, 150), (4, 23)]


def _stats(cf, monkeypatch, split, cfg, y, init, lat, **kw):
    monkeypatch.setenv("CFUST_SPLIT", str(split))
    em = cf.CfustEM(y, cfg.g, cfg.q, init, lat, **kw)
    ll, st = em.estep(want_stats=True)
    em.close()
    return ll, st


@pytest.mark.parametrize("cfg_id,n", CASES)
@pytest.mark.parametrize("split", [1, 2, 4, 8])
def test_split_stats_parity(cf, orc, monkeypatch, cfg_id, n, split):
    cfg, y, init, lat = _problem(cfg_id, n)
    ll, st = _stats(cf, monkeypatch, split, cfg, y, init, lat)
    ref = orc.estep(y, init, cfg.q, _olat(orc, lat))
    compare_stats(st, ref["stats"], cfg.p, cfg.q, cfg.g)
    assert abs(ll - ref["loglik"]) <= TOL * abs(ref["loglik"])


@pytest.mark.parametrize("cfg_id,n", CASES)
def test_split_agrees_with_one_warp(cf, monkeypatch, cfg_id, n):
    cfg, y, init, lat = _problem(cfg_id, n)
    ll1, st1 = _stats(cf, monkeypatch, 1, cfg, y, init, lat)
    for split in (2, 4, 8):
        ll, st = _stats(cf, monkeypatch, split, cfg, y, init, lat)
        assert abs(ll - ll1) <= 1e-13 * abs(ll1)
        np.testing.assert_allclose(st, st1, rtol=1e-12, atol=1e-12 * np.abs(st1).max())


def test_split_exact_e1(cf, orc, monkeypatch):
    """T_eval_w (exact e1, reading R2') under SPLIT: the f-weighted log V sum is split as well."""
    import synth
    cfg, y, init, _ = _problem(5, 120)
    lat = synth.lattice_inputs(cfg, e1_exact=True)
    ll, st = _stats(cf, monkeypatch, 4, cfg, y, init, lat, e1_exact=True)
    ref = orc.estep(y, init, cfg.q, _olat(orc, lat), e1_exact=True)
    compare_stats(st, ref["stats"], cfg.p, cfg.q, cfg.g)


def test_split_fit_parity(cf, orc, monkeypatch):
    cfg, y, init, lat = _problem(1, 202)   # AIS-sized n, q = p = 2
    monkeypatch.setenv("CFUST_SPLIT", "8")
    em = cf.CfustEM(y, cfg.g, cfg.q, init, lat)
    res = em.fit(10)
    em.close()
    ref = orc.fit(y, init, cfg.q, _olat(orc, lat), max_iter=10)
    assert np.max(np.abs(res["trace"] - ref["trace"]) / np.abs(ref["trace"])) <= TOL
