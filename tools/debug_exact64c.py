import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_1403_7458_b200 as sp
from oracle import spamm_oracle as O
from conftest import golden, pyramid_flat
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[4]
h, n_occ = water_cluster(cfg.n_mol, seed=0)
f = sp.build_from_dense(h, 64); of = O.from_dense(h, 64)
x = sp.sp2_init(f, sp.gershgorin_bounds(f)); ox = O.sp2_init(of, O.gershgorin_bounds(of))
def cmp(tag, a, oa):
    d, od = sp.to_dense(a), O.to_dense(oa)
    ok = np.array_equal(d, od) and np.array_equal(pyramid_flat(a._tier_norms), pyramid_flat(oa.tier_norms)) and np.array_equal(a._block_keys, oa.keys)
    if not ok:
        idx = np.argwhere(d != od)
        print(tag, "DIFF", len(idx), idx[:4], "stored", a.stored_leaf_count, len(oa.keys), flush=True)
        if len(idx): print("  vals", d[tuple(idx[0])], od[tuple(idx[0])])
    return ok
for it in range(36):
    c, st = sp.multiply(x, x, cfg.tau, kernel="exact")
    oc, ost, _ = O.multiply(ox, ox, cfg.tau, threads=16)
    if not cmp(f"{it} X2", c, oc): break
    tx, tq = sp.trace(x), sp.trace(c)
    idem = sp.add_scaled(1.0, c, -1.0, x); oidem = O.add_scaled(1.0, oc, -1.0, ox)
    if not cmp(f"{it} idem", idem, oidem): break
    e, oe = idem.norm(), oidem.norm()
    br = abs(tq - n_occ) <= abs(2 * tx - tq - n_occ)
    print(it, "ok", br, e == oe, e, flush=True)
    if br: x, ox = c, oc
    else:
        x = sp.add_scaled(2.0, x, -1.0, c); ox = O.add_scaled(2.0, ox, -1.0, oc)
        if not cmp(f"{it} expand", x, ox): break
