"""N > 1 host logic on CPU with world_size-2 gloo process groups: shard partitioning, the
ncclUniqueId broadcast helper, and the algebra of one all-reduce of the sufficient statistics
per iteration followed by the replicated M-step (Alg. 2-3).  The E-step /
M-step arithmetic here is the oracle's (CUDA kernels need a GPU); the sharding, the exchange
and the max-over-ranks timing are the product's code (paper_2005_06848_b200.dist), driven through
the same bootstrap / Ranks calls bench.py makes."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import oracle
    import synth as S
    from paper_2005_06848_b200 import dist as D
    # the torchrun environment bench.py reads (D.env_rank), then bench.py's own bootstrap
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank)})
    rk = D.bootstrap("gloo")
    try:
        assert (rk.rank, rk.world, rk.device) == (rank, world, "cpu")
        uid = rk.nccl_id(make_id=lambda: bytes(range(128)))          # what every CfustEM context receives
        assert uid == bytes(range(128))
        cfg = S.with_n(S.CONFIGS[1], 301)
        y, init, _ = S.make_problem(cfg)
        M, z, sh = S.lattice_inputs(cfg)
        lat = oracle.Lattice(M, z, sh)
        j0, j1 = rk.shard(cfg.n)
        assert (j0, j1) == S.shard_range(cfg.n, rank, world)
        params = init
        trace = []
        for it in range(3):
            st = oracle.estep(y[j0:j1], params, cfg.q, lat, nthreads=1)["stats"]
            # the exchanged vector: [statistics, l, underflow flag], summed by the ONE all-reduce
            v = np.concatenate([st, [0.0]])
            t = torch.from_numpy(v.copy())
            rk.dist.all_reduce(t)                                  # the one exchange per iteration
            assert float(t[-1]) == 0.0                             # no rank underflowed
            trace.append(float(t[-2]))
            rc, params = oracle.mstep(t.numpy()[:-1], params, cfg.p, cfg.q, cfg.n)
            assert rc == 0
        rk.barrier()
        tmax = rk.max(1.0 + rank)                                  # bench.py's max-over-ranks timing
        assert tmax == float(world)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), trace=np.array(trace), **params)
    finally:
        rk.close()


@pytest.mark.parametrize("world", [2])
def test_two_rank_em_equals_single(tmp_path, world):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    import oracle
    oracle.build()
    cfg = synth.with_n(synth.CONFIGS[1], 301)
    y, init, _ = synth.make_problem(cfg)
    M, z, sh = synth.lattice_inputs(cfg)
    lat = oracle.Lattice(M, z, sh)
    params, trace = init, []
    for it in range(3):
        out = oracle.estep(y, params, cfg.q, lat, nthreads=1)
        trace.append(out["loglik"])
        rc, params = oracle.mstep(out["stats"], params, cfg.p, cfg.q, cfg.n)
    r = [np.load(tmp_path / f"r{k}.npz") for k in range(world)]
    for k in range(1, world):                                 # replicas stay identical
        for key in ["pi", "mu", "sigma", "delta", "nu"]:
            assert np.array_equal(r[0][key], r[k][key])
    assert np.max(np.abs(r[0]["trace"] - np.array(trace)) / np.abs(trace)) < 1e-12
    for key in ["pi", "mu", "sigma", "delta", "nu"]:
        assert np.max(np.abs(r[0][key] - params[key])) <= 1e-10 * max(1.0, np.max(np.abs(params[key])))


def test_shard_range_properties():
    from paper_2005_06848_b200.dist import shard_range
    for n in [0, 1, 7, 100_001]:
        for w in [1, 2, 3, 8]:
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[k][1] == rs[k + 1][0] for k in range(w - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
