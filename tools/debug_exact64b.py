import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_1403_7458_b200 as sp
from conftest import golden, pyramid_flat
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
gd = golden("cfg4_sp2"); cfg = CONFIGS[4]
h, n_occ = water_cluster(cfg.n_mol, seed=0)
f = sp.build_from_dense(h, 64)
for kern in ("exact", "auto", "exact"):
    pe, ste = sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro", fro_tol=1e-6, kernel=kern)
    t = np.array(ste.trace_history); g = gd["traces"]
    print(kern, ste.iteration, len(t), np.flatnonzero(t != g)[:10], (t - g)[t != g][:5],
          "idem", np.array_equal(np.array(ste.idempotency_history), gd["idem"]),
          "p", np.array_equal(pyramid_flat(pe._tier_norms), gd["p_pyramid"]), flush=True)
