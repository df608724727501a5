import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from oracle import spamm_oracle as O
from conftest import golden, pyramid_flat
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
gd = golden('cfg4_sp2'); cfg = CONFIGS[4]
h, n_occ = water_cluster(cfg.n_mol, seed=0)
print("h checksum", float(np.abs(h).sum()), h[5, 7], flush=True)
f = O.from_dense(h, 64)
print("f pyr", np.array_equal(pyramid_flat(f.tier_norms), gd["f_pyramid"]), flush=True)
for thr in (8, 16):
    res = O.sp2_solve(f, n_occ, cfg.tau, threads=thr, criterion='fro')
    t = np.array(res.trace_history); g = gd['traces']
    print(thr, res.iterations, np.flatnonzero(t != g)[:10], flush=True)
