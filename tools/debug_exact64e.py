import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_1403_7458_b200 as sp
from conftest import golden, pyramid_flat
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
from paper_1403_7458_b200 import sp2 as S
gd = golden("cfg4_sp2"); cfg = CONFIGS[4]
h, n_occ = water_cluster(cfg.n_mol, seed=0)
f = sp.build_from_dense(h, 64)
# instrumented copy of sp2_solve
x = S.sp2_init(f, S.gershgorin_bounds(f))
xs_a = []
for it in range(30):
    x_next, branch, t_x, t_sq, stats, x_sq = S._step(x, n_occ, cfg.tau, "serial", None, "exact")
    idem = S.add_scaled(1.0, x_sq, -1.0, x).norm()
    if branch == S.EXPAND:
        x_next = S.add_scaled(2.0, x, -1.0, x_sq)
    x = x_next
    xs_a.append((sp.trace(x), branch, stats.leaf_products, x.stored_leaf_count, sp.to_dense(x)))
# lockstep version
x = S.sp2_init(f, S.gershgorin_bounds(f))
for it in range(30):
    c, st = sp.multiply(x, x, cfg.tau, kernel="exact")
    tx, tq = sp.trace(x), sp.trace(c)
    br = abs(tq - n_occ) <= abs(2 * tx - tq - n_occ)
    x = c if br else sp.add_scaled(2.0, x, -1.0, c)
    ta, bra, lpa, sta, da = xs_a[it]
    db = sp.to_dense(x)
    print(it, ta == sp.trace(x), bra, br, lpa, st.leaf_products, sta, x.stored_leaf_count, np.array_equal(da, db), float(gd["traces"][it + 1]) == ta, flush=True)
