"""Debug: locate skew-normal pairs with non-finite e3/e4 on full cfg5 and compare with the oracle."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import synth, paper_2005_06848_b200 as cf
import oracle as orc
cfg = synth.CONFIGS[5]
y, init, _ = synth.make_problem(cfg)
yd = torch.from_numpy(y).cuda()
lat = synth.lattice_inputs(cfg)
em = cf.CfustEM(yd, cfg.g, cfg.q, init, lat, family="sn")
bad = []
for j0 in range(0, cfg.n, 500000):
    idx = np.arange(j0, min(cfg.n, j0 + 500000))
    pr = em.pairs(idx)
    nf = ~np.isfinite(pr[:, :, 4:]).all(axis=2)
    for jj, i in zip(*np.nonzero(nf)):
        bad.append((int(idx[jj]), int(i), pr[jj, i]))
print("bad pairs:", len(bad))
for j, i, row in bad[:6]:
    print("j", j, "comp", i, "gpu row", row)
    ref = orc.estep(y[j:j + 1], init, cfg.q, orc.Lattice(*lat), pairs=True, family="sn")["pairs"][0, i]
    print("   oracle row", ref)
