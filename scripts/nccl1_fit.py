"""A cfust_fit on a one-rank NCCL communicator (world = 1 with an ncclUniqueId: every collective path
live) — run under `ncu --metrics gpu__time_duration.sum` to show the launch sequence of an EM
iteration: E-step kernel, reduce, ONE ncclAllReduce kernel, M-step, chi nodes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2005_06848_b200 as cf  # noqa: E402

cfg = synth.with_n(synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1], 1000)
y, init, _ = synth.make_problem(cfg)
em = cf.CfustEM(y, cfg.g, cfg.q, init, synth.lattice_inputs(cfg), world=1, rank=0, nccl_id=cf.nccl_unique_id())
r = em.fit(4)
print("fit", r["n_iter"], r["trace"][-1], "launches", em.launch_count)
em.close()
