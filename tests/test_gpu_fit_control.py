"""cfust_fit control flow on the GPU (a10 + the graph-captured iteration):

- tol > 0: the Aitken rule (Alg. 4; reading A8) stops the GPU fit at the same
  iteration as the oracle's orc_fit, with the same `converged` flag and trace (1e-9) — default,
  SOV-direct and q = 0 contexts;
- the last trace entry equals a fresh cfust_estep's l bit for bit (the final density pass);
- the CUDA-graph path (default) and the eager path (timing contexts) give identical bits;
- transactional M-step: a failing component (EEMPTY) or an E-step underflow leaves Psi^(k) of every
  component untouched."""
import numpy as np
import pytest

import synth
from test_gpu_parity import PTOL, TOL, _olat, _problem, compare_params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_06848_b200 import build as B
    B.build()
    import paper_2005_06848_b200 as m
    return m


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.build()
    return oracle


def _lat_for(cfg, opt):
    return synth.lattice_inputs(cfg, e1_exact=opt.get("e1_exact", False), direct=opt.get("estimator") == "direct")


# tolerances chosen so that the rule fires well inside max_iter and away from its threshold
# (oracle: stops at k = 13, 2, 3, 2, 8; |l_inf - l_k| stays >= 11 % away from tol at every k)
@pytest.mark.parametrize("cfg_id,n,tol,opt", [(1, 1000, 1e-2, {}), (2, 150, 2.0, {}), (3, 20000, 1e-1, {}),
                                              (5, 200, 5.0, {"estimator": "direct"}), (1, 1000, 2.6, {"family": "sn"})])
def test_fit_aitken_matches_oracle(cf, orc, cfg_id, n, tol, opt):
    cfg, y, init, _ = _problem(cfg_id, n)
    lat = _lat_for(cfg, opt)
    em = cf.CfustEM(y, cfg.g, cfg.q, init, lat, **opt)
    res = em.fit(60, tol)
    ref = orc.fit(y, init, cfg.q, _olat(orc, lat), max_iter=60, tol=tol, **opt)
    assert ref["rc"] == 0
    assert ref["converged"] and ref["n_iter"] < 60, "pick a tolerance the rule reaches"
    assert res["n_iter"] == ref["n_iter"] and res["converged"] == ref["converged"]
    assert np.max(np.abs(res["trace"] - ref["trace"]) / np.abs(ref["trace"])) <= TOL
    compare_params(res["params"], ref["params"], cfg.q, tol=PTOL)
    em.close()


@pytest.mark.parametrize("cfg_id,n,opt", [(2, 300, {}), (5, 500, {"estimator": "direct"}), (3, 5000, {})])
def test_fit_last_l_equals_estep(cf, cfg_id, n, opt):
    cfg, y, init, _ = _problem(cfg_id, n)
    lat = _lat_for(cfg, opt)
    em = cf.CfustEM(y, cfg.g, cfg.q, init, lat, **opt)
    res = em.fit(4)
    assert res["n_iter"] == 4 and len(res["trace"]) == 5
    assert res["trace"][-1] == em.estep()          # bit-identical l at the final Psi
    em.close()


@pytest.mark.parametrize("cfg_id,n", [(1, 1000), (5, 400), (3, 3000)])
def test_graph_equals_eager(cf, cfg_id, n):
    """timing=True contexts run the eager launch sequence; default contexts the captured graphs."""
    cfg, y, init, lat = _problem(cfg_id, n)
    a = cf.CfustEM(y, cfg.g, cfg.q, init, lat)
    b = cf.CfustEM(y, cfg.g, cfg.q, init, lat, timing=True)
    for _ in range(2):
        assert a.iterate() == b.iterate()
    ra, rb = a.fit(3), b.fit(3)
    assert np.array_equal(ra["trace"], rb["trace"])
    for k in ra["params"]:
        assert np.array_equal(ra["params"][k], rb["params"][k])
    ra, rb = a.fit(5, 1e-3), b.fit(5, 1e-3)
    assert ra["n_iter"] == rb["n_iter"] and np.array_equal(ra["trace"], rb["trace"])
    a.close()
    b.close()


def test_long_fit_drains_trace_ring(cf, orc):
    """A fit longer than the device trace ring (4096 slots) keeps every l^(k) (q = 0, tiny n)."""
    cfg, y, init, lat = _problem(3, 64)
    em = cf.CfustEM(y, cfg.g, cfg.q, init, lat)
    res = em.fit(4200)
    assert res["n_iter"] == 4200 and len(res["trace"]) == 4201 and np.all(np.isfinite(res["trace"]))
    ref = orc.fit(y, init, 0, None, max_iter=30)
    assert np.max(np.abs(res["trace"][:31] - ref["trace"]) / np.abs(ref["trace"])) <= TOL
    em.close()


def _params_equal(a, b):
    return all(np.array_equal(a[k], b[k]) for k in a)


def test_mstep_empty_component_leaves_psi_unchanged(cf):
    """Component 1 sits far from every observation with a tiny weight: S0_1 < 1e-10 -> EEMPTY.
    No component's parameters move (the M-step commits only after every component succeeded)."""
    cfg, y, init, lat = _problem(1, 400)
    bad = {k: np.array(v, dtype=np.float64, copy=True) for k, v in init.items()}
    bad["mu"][1] = bad["mu"][1] + 1e3
    bad["pi"] = np.array([1.0 - 1e-12, 1e-12])
    em = cf.CfustEM(y, cfg.g, cfg.q, bad, lat)
    before = em.params()
    em.estep()
    with pytest.raises(cf.CfustError) as e:
        em.mstep()
    assert e.value.code == cf.CFUST_EEMPTY
    assert _params_equal(before, em.params())
    with pytest.raises(cf.CfustError) as e:
        em.fit(3)
    assert e.value.code == cf.CFUST_EEMPTY
    assert _params_equal(before, em.params())
    em.close()


def test_underflow_gates_mstep(cf):
    """An E-step underflow (every component density 0 at some y_j, A16) stops the fit with
    EUNDERFLOW and Psi unchanged (the M-step gates itself on the flag carried by the all-reduce)."""
    params = {"pi": [1.0], "mu": [[0.0]], "sigma": [[[1e-4]]], "delta": [[[5.0]]], "nu": [1000.0]}
    em = cf.CfustEM(np.array([[-1e4], [0.1], [0.2]]), 1, 1, params, None)
    before = em.params()
    with pytest.raises(cf.CfustError) as e:
        em.iterate()
    assert e.value.code == cf.CFUST_EUNDERFLOW
    assert _params_equal(before, em.params())
    with pytest.raises(cf.CfustError) as e:
        em.fit(3)
    assert e.value.code == cf.CFUST_EUNDERFLOW
    assert _params_equal(before, em.params())
    em.close()
