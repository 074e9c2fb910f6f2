"""The oracle's parity-harness outputs (tests only): the running error bounds of e3 / e4
(reading P1) and the reversed near-tie order (reading A14).  Neither may change the E-step."""
import numpy as np
import pytest

import synth


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.build()
    return oracle


def _setup(cfg_id, n, **kw):
    cfg = synth.with_n(synth.CONFIGS[cfg_id], n)
    if kw:
        cfg = synth.with_(cfg, **kw)
    y, init, _ = synth.make_problem(cfg)
    return cfg, y, init, synth.lattice_inputs(cfg)


@pytest.mark.parametrize("cfg_id,family", [(1, "st"), (2, "st"), (2, "sn")])
def test_bounds_dominate_moments_and_leave_estep_unchanged(orc, cfg_id, family):
    cfg, y, init, lat = _setup(cfg_id, 40)
    L = orc.Lattice(*lat)
    a = orc.estep(y, init, cfg.q, L, pairs=True, bounds=True, family=family)
    b = orc.estep(y, init, cfg.q, L, pairs=True, family=family)
    assert np.array_equal(a["pairs"], b["pairs"]) and np.array_equal(a["stats"], b["stats"])
    q = cfg.q
    B = a["bounds"]
    e3, e4 = a["pairs"][..., 4:4 + q], a["pairs"][..., 4 + q:]
    fin = np.isfinite(a["pairs"][..., 0])
    # a sum's running bound (sum of |terms|) is >= |sum|
    assert np.all(B[..., :q][fin] >= np.abs(e3[fin]) * (1 - 1e-12))
    assert np.all(B[..., q:][fin] >= np.abs(e4[fin]) * (1 - 1e-12))


def test_bounds_grow_in_the_deep_tail(orc):
    """Reading P1: for an observation far in a component's tail (alpha = c / sqrt(S') << 0) the
    bound / |e4| ratio (the condition number of E2) is large; near the mode it is O(1)."""
    cfg, y, init, lat = _setup(1, 10)
    L = orc.Lattice(*lat)
    mu0 = np.asarray(init["mu"][0])
    rc, dv = orc.derive(init["sigma"][0], init["delta"][0], init["nu"][0])
    A, sl = dv["A"], np.sqrt(np.diag(dv["Lambda"]))
    # y = mu + r with c = A r = alpha sqrt(diag Lambda): alpha = 0.3 (mode side) and -8 (deep tail)
    yy = np.stack([mu0 + np.linalg.pinv(A) @ (al * sl) for al in (0.3, -8.0)])
    a = orc.estep(yy, init, 2, L, pairs=True, bounds=True, family="sn")
    e4 = np.max(np.abs(a["pairs"][:, 0, 6:]), axis=-1)
    cond = np.max(a["bounds"][:, 0, 2:], axis=-1) / e4
    assert cond[0] < 10.0 and cond[1] > 1e3, cond


def test_tie_flip_only_moves_near_tied_pairs(orc):
    """y = mu + Delta u with Lambda's symmetric structure gives exact key ties (c_k equal): the
    flipped order changes T only at the QMC level; pairs without near ties are bit-identical."""
    cfg, y, init, lat = _setup(1, 30)
    L = orc.Lattice(*lat)
    a = orc.estep(y, init, cfg.q, L, pairs=True, gaps=True)
    b = orc.estep(y, init, cfg.q, L, pairs=True, gaps=True, tie_flip=True)
    near = a["gaps"] <= 1e-12
    same = np.all(a["pairs"] == b["pairs"], axis=-1)
    # tau couples the components of an observation: compare rows without any near tie
    rows = ~np.any(near, axis=1)
    assert np.all(same[rows])
    # an exact tie: c = 0 (y on the Omega-orthogonal complement of Delta) gives equal keys 0
    mu0 = np.asarray(init["mu"][0])
    yt = mu0[None, :].copy()                     # r = 0 -> c = 0 for component 0
    a = orc.estep(yt, init, cfg.q, L, pairs=True, gaps=True)
    b = orc.estep(yt, init, cfg.q, L, pairs=True, gaps=True, tie_flip=True)
    assert a["gaps"][0, 0] == 0.0
    d = np.abs(a["pairs"][0, 0] - b["pairs"][0, 0]) / np.maximum(np.abs(a["pairs"][0, 0]), 1e-300)
    assert np.max(d) < 1e-3          # both orders estimate the same integrals (QMC error level)
