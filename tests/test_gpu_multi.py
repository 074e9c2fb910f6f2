"""Two ranks on two GPUs (skipped unless torch.cuda.device_count() >= 2; the round-end GPU boxes of
this project have one): each rank builds a context on its contiguous shard with a shared
ncclUniqueId, runs an E-step (ONE all-reduce of [statistics, l, flag]) and a 3-iteration fit; the
all-reduced statistics and the fitted parameters must equal the single-GPU context's (sums in a
different order: 1e-12), and both ranks must hold bit-identical parameters (replicated M-step)."""
import os
import socket

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank)})
    import synth as S
    import paper_2005_06848_b200 as cf
    from paper_2005_06848_b200 import dist as D
    rk = D.bootstrap("nccl")
    try:
        cfg = S.with_n(S.CONFIGS[5], 3001)
        y, init, _ = S.make_problem(cfg)
        j0, j1 = rk.shard(cfg.n)
        em = cf.CfustEM(y[j0:j1], cfg.g, cfg.q, init, S.lattice_inputs(cfg), n_total=cfg.n, rank=rank, world=world,
                        nccl_id=rk.nccl_id(), device=rk.local, global_offset=j0)
        ll, st = em.estep(want_stats=True)
        res = em.fit(3)
        np.savez(os.path.join(out_dir, f"g{rank}.npz"), st=st, trace=res["trace"], **res["params"])
        em.close()
    finally:
        rk.close()


def test_two_gpu_allreduce_and_fit(tmp_path):
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import torch.multiprocessing as mp
    mp.spawn(_rank, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    import paper_2005_06848_b200 as cf
    cfg = synth.with_n(synth.CONFIGS[5], 3001)
    y, init, _ = synth.make_problem(cfg)
    one = cf.CfustEM(y, cfg.g, cfg.q, init, synth.lattice_inputs(cfg))
    _, st = one.estep(want_stats=True)
    ref = one.fit(3)
    r = [np.load(tmp_path / f"g{k}.npz") for k in range(2)]
    assert np.array_equal(r[0]["st"], r[1]["st"])
    assert np.max(np.abs(r[0]["st"] - st) / np.maximum(np.abs(st), 1e-300)) < 1e-12
    for key in ["pi", "mu", "sigma", "delta", "nu"]:
        assert np.array_equal(r[0][key], r[1][key])                       # replicated M-step
        a, b = r[0][key], np.asarray(ref["params"][key])
        assert np.max(np.abs(a - b)) <= 1e-10 * max(1.0, np.max(np.abs(b)))
    assert np.max(np.abs(r[0]["trace"] - ref["trace"]) / np.abs(ref["trace"])) < 1e-12
    one.close()
