"""The NCCL code paths on one GPU: a context with world = 1 and an ncclUniqueId runs every
collective (the statistics all-reduce, the status agreement, Alg. 1's all-reduces and all-gather)
over a one-rank communicator; results must equal the context without NCCL bit for bit."""
import numpy as np
import pytest

import synth

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


@pytest.mark.parametrize("cfg_id,n", [(1, 1000), (3, 5000), (5, 400)])
def test_one_rank_nccl_equals_no_nccl(cf, cfg_id, n):
    cfg = synth.with_n(synth.CONFIGS[cfg_id], n)
    y, init, _ = synth.make_problem(cfg)
    lat = synth.lattice_inputs(cfg)
    a = cf.CfustEM(y, cfg.g, cfg.q, init, lat)
    b = cf.CfustEM(y, cfg.g, cfg.q, init, lat, world=1, rank=0, nccl_id=cf.nccl_unique_id())
    la, sa = a.estep(want_stats=True)
    lb, sb = b.estep(want_stats=True)
    assert la == lb and np.array_equal(sa, sb)
    ra, rb = a.fit(3), b.fit(3)
    assert np.array_equal(ra["trace"], rb["trace"])
    for k in ra["params"]:
        assert np.array_equal(ra["params"][k], rb["params"][k])
    pa = a.init_partitions(4, seed=11)
    pb = b.init_partitions(4, seed=11)
    assert np.array_equal(pa, pb)
    (lla0, besta), (llb0, bestb) = a.init_select(4), b.init_select(4)
    assert besta == bestb and np.array_equal(lla0, llb0)
    la_, ta, lla = a.predict()
    lb_, tb, llb = b.predict()
    assert np.array_equal(la_, lb_) and np.array_equal(ta, tb) and lla == llb
    a.close()
    b.close()


def test_collective_wait_timeout_fails_fast(cf, monkeypatch):
    """Failure detection: with CFUST_NCCL_TIMEOUT_S below one E-step's duration the NCCL-aware wait
    aborts the communicator and returns CFUST_ENCCL; every later call on the context fails the
    same way (no silent fallback to single-rank semantics)."""
    cfg = synth.with_n(synth.CONFIGS[2], 2000)
    y, init, _ = synth.make_problem(cfg)
    em = cf.CfustEM(y, cfg.g, cfg.q, init, synth.lattice_inputs(cfg), world=1, rank=0,
                    nccl_id=cf.nccl_unique_id())
    em.estep()                                        # healthy first
    monkeypatch.setenv("CFUST_NCCL_TIMEOUT_S", "1e-9")   # read at every collective wait
    with pytest.raises(cf.CfustError) as e:
        em.estep()
    assert e.value.code == cf.CFUST_ENCCL
    monkeypatch.delenv("CFUST_NCCL_TIMEOUT_S")
    with pytest.raises(cf.CfustError) as e2:
        em.loglik()
    assert e2.value.code == cf.CFUST_ENCCL
    em.close()
