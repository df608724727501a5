"""Bisect the nondeterminism of the cfg3 SP2 solve over feature switches."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[3]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(h, cfg.block_size)


def run(label, reps=8, **kw):
    ref, bad = None, 0
    for _ in range(reps):
        p, st = sp.sp2_solve(f, n_occ, cfg.tau, **kw)
        d = sp.to_dense(p)
        if ref is None:
            ref = d
        elif not np.array_equal(d, ref):
            bad += 1
    print(f"{label:40s} nondeterministic runs: {bad}/{reps - 1}", flush=True)


mode = sys.argv[1]
if mode == "fro":
    run("fro (fused residual + union)", criterion="fro", fro_tol=1e-6)
elif mode == "trace":
    run("trace criterion", criterion="trace")
elif mode == "walk":
    sp.set_dense_cull(False)
    run("fro, tier-walk cull", criterion="fro", fro_tol=1e-6)
elif mode == "nosym":
    sp.set_symmetric_products(False)
    run("fro, no symmetric products", criterion="fro", fro_tol=1e-6)
