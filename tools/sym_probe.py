"""Is X^2 exactly symmetric for exactly symmetric X (DMMA and exact kernels)?"""
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
for ci in (3, 4):
    cfg = CONFIGS[ci]
    h, n_occ = water_cluster(cfg.n_mol, seed=0)
    f = sp.build_from_dense(h, cfg.block_size)
    x = sp.sp2_init(f, sp.gershgorin_bounds(f))
    d = sp.to_dense_device(x)
    print(cfg.name, "X0 symmetric", torch.equal(d, d.T))
    for kern in ("dmma", "exact"):
        xx = x
        for it in range(6):
            c, st = sp.multiply(xx, xx, cfg.tau, kernel=kern)
            dc = sp.to_dense_device(c)
            print(" ", kern, it, "C==C^T", torch.equal(dc, dc.T), "ndiff", int((dc != dc.T).sum()))
            xx = c
