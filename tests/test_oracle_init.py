"""Pins for the oracle's Alg. 1 (parallel multi-start initialisation; NEXT-1)
under readings I1-I4: random partitions, k-means, Psi^(0) from a partition,
candidate selection.  References: scikit-learn's Lloyd k-means, numpy moments, the E-step."""
import numpy as np
import pytest
import scipy.stats as st

import synth


def test_random_partition_properties(orc):
    """I1: labels in [0, g), >= p+1 members, deterministic, uniform (chi-square), independent
    across candidates (agreement ~ 1/g); SPEC.md:414 infeasible example."""
    n, p, g = 100_000, 3, 5
    a, lab = orc.random_partition(n, p, g, 1234, 1, 8)
    assert a == 0 and lab.min() >= 0 and lab.max() < g
    assert np.array_equal(lab, orc.random_partition(n, p, g, 1234, 1, 8)[1])
    cnt = np.bincount(lab, minlength=g)
    chi2 = ((cnt - n / g) ** 2 / (n / g)).sum()
    assert chi2 < st.chi2.ppf(0.999, g - 1), cnt
    _, lab2 = orc.random_partition(n, p, g, 1234, 2, 8)
    agree = (lab == lab2).mean()
    assert abs(agree - 1 / g) < 5 * np.sqrt((1 / g) * (1 - 1 / g) / n)
    _, lab3 = orc.random_partition(n, p, g, 99, 1, 8)
    assert abs((lab == lab3).mean() - 1 / g) < 0.01
    assert orc.random_partition(4, 3, 2, 1, 1, 2)[0] == orc.EINVAL      # needs >= 8 points
    # small n: the attempt loop redraws until every component has p+1 members
    a, lab = orc.random_partition(12, 2, 4, 7, 1, 2)
    assert a >= 0 and np.bincount(lab, minlength=4).min() >= 3


def _farthest_point_centres(y, g, seed, orc):
    """Reading I2 seeding written out with numpy (independent of the oracle's loop)."""
    n = len(y)
    j0 = orc.splitmix64(seed ^ 0xA5A5A5A5A5A5A5A5) % n
    cen = [y[j0]]
    mind = ((y - y[j0]) ** 2).sum(1)
    for _ in range(1, g):
        j = int(np.argmax(mind))          # numpy argmax: first maximal index
        cen.append(y[j])
        mind = np.minimum(mind, ((y - y[j]) ** 2).sum(1))
    return np.array(cen)


@pytest.mark.parametrize("cfg_id,n", [(1, 3000), (5, 20000), (3, 8000)])
def test_kmeans_vs_sklearn_lloyd(orc, cfg_id, n):
    """I2: from the same farthest-point centres, the oracle's Lloyd fixed point equals
    scikit-learn's Lloyd k-means (n_init=1, tol=0) label for label; centres are the member means."""
    from sklearn.cluster import KMeans
    cfg = synth.with_n(synth.CONFIGS[cfg_id], n)
    y, _, _ = synth.make_problem(cfg)
    rc, lab, cen = orc.kmeans(y, cfg.g, 2024, 300)
    assert rc == 0
    init = _farthest_point_centres(y, cfg.g, 2024, orc)
    km = KMeans(cfg.g, init=init, n_init=1, max_iter=300, tol=0.0, algorithm="lloyd").fit(y)
    assert np.array_equal(lab, km.labels_)
    for i in range(cfg.g):
        assert np.allclose(cen[i], y[lab == i].mean(0), rtol=1e-12, atol=1e-12)
    d = ((y[:, None, :] - cen[None]) ** 2).sum(2)
    assert np.array_equal(lab, d.argmin(1))


def test_kmeans_separates_blobs(orc):
    """two obvious blobs at +-10 with unit noise, g = 2 -> exact separation."""
    rng = np.random.default_rng(0)
    y = np.concatenate([rng.standard_normal((500, 2)) - 10, rng.standard_normal((500, 2)) + 10])
    rc, lab, _ = orc.kmeans(y, 2, 5, 50)
    assert rc == 0
    assert len(set(lab[:500])) == 1 and len(set(lab[500:])) == 1 and lab[0] != lab[-1]


@pytest.mark.parametrize("q", [0, 2, 3])
def test_partition_params_vs_numpy(orc, q):
    """I3 against numpy moments: pi, ybar, biased covariance, skewness sign, Delta, mu, nu."""
    cfg = synth.with_(synth.with_n(synth.CONFIGS[1], 4000), q=q, p=3, g=3)
    y, _, truth = synth.make_problem(cfg)
    _, lab = orc.random_partition(len(y), cfg.p, cfg.g, 77, 1, 4)
    rc, P = orc.partition_params(y, lab, cfg.g, q)
    assert rc == 0
    for i in range(cfg.g):
        yi = y[lab == i]
        S = np.cov(yi.T, bias=True)
        assert abs(P["pi"][i] - len(yi) / len(y)) < 1e-15
        assert np.allclose(P["sigma"][i], S, rtol=1e-11, atol=1e-12)
        D = np.zeros((cfg.p, q))
        sk = st.skew(yi, axis=0)
        for k in range(min(cfg.p, q)):
            D[k, k] = (0.5 if sk[k] >= 0 else -0.5) * np.sqrt(S[k, k])
        assert np.allclose(P["delta"][i], D, rtol=1e-11, atol=1e-12)
        assert np.allclose(P["mu"][i], yi.mean(0) - np.sqrt(2 / np.pi) * D.sum(1), rtol=1e-11, atol=1e-12)
        assert P["nu"][i] == 10.0
    bad = np.zeros(len(y), np.int32)                    # components 1, 2 empty -> invalid
    assert orc.partition_params(y, bad, cfg.g, q)[0] == orc.EINVAL


def test_init_select_is_argmax_of_estep_loglik(orc):
    """I4: loglik0[c] is the E-step log-likelihood at Psi^(0)_c (definition, Eq. (3)); the winner
    is the argmax (reading A9: largest), and with the true labels among random candidates on
    well-separated data the true partition wins."""
    cfg = synth.with_(synth.with_n(synth.CONFIGS[1], 1500), p=2, q=2, g=2)
    truth = synth.make_truth(cfg)
    truth["mu"] = truth["mu"] * 4.0                     # well separated
    y, labels = synth.sample(cfg, truth, return_labels=True)
    M, z, sh = synth.lattice_inputs(cfg)
    lat = orc.Lattice(M, z, sh)
    cands = [orc.random_partition(len(y), cfg.p, cfg.g, 5, l, 4)[1] for l in range(1, 4)]
    cands.insert(2, labels.astype(np.int32))
    res = orc.init_select(y, np.array(cands), cfg.g, cfg.q, lat)
    assert res["rc"] == 0 and res["best"] == 2
    for c in range(4):
        _, P = orc.partition_params(y, cands[c], cfg.g, cfg.q)
        assert res["loglik0"][c] == orc.estep(y, P, cfg.q, lat)["loglik"]
    assert res["loglik0"][2] == res["loglik0"].max()
    # burn-in: the winner's l after r EM iterations is the fit's l^(r)
    rb = orc.init_select(y, np.array(cands), cfg.g, cfg.q, lat, burn_in=2)
    _, P = orc.partition_params(y, cands[rb["best"]], cfg.g, cfg.q)
    assert rb["loglik0"][rb["best"]] == orc.fit(y, P, cfg.q, lat, max_iter=2)["trace"][-1]
