import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import synth, paper_2005_06848_b200 as cf
cfg = synth.CONFIGS[3]
y, init, _ = synth.make_problem(cfg)
yd = torch.from_numpy(y).cuda()
em = cf.CfustEM(yd, cfg.g, 0, init, None, timing=True)
for _ in range(3): em.estep(); em.loglik()
torch.cuda.synchronize()
s = torch.cuda.ExternalStream(em.stream_ptr)
for name, fn in [("estep", em.estep), ("loglik", em.loglik)]:
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(20): fn()
    e1.record(s); e1.synchronize()
    print(name, e0.elapsed_time(e1) / 20, "ms per call (incl. reduce + sync)")
