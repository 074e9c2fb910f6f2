import sys, os
sys.path.insert(0, os.getcwd())
import synth, paper_2005_06848_b200 as cf
for c in (1, 3):
    cfg = synth.CONFIGS[c]
    y, init, _ = synth.make_problem(cfg)
    em = cf.CfustEM(y, cfg.g, cfg.q, init, synth.lattice_inputs(cfg), timing=True)
    for _ in range(3):
        em.iterate()
    print("cfg", c, flush=True)
    em.iterate()
    em.close()
